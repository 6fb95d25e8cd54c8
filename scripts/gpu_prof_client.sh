#!/bin/bash
# ncu of the client-side kernels (decryption scaling, encryption prep) inside the e2e breakdown script
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python scripts/e2e_parts.py > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none -k 'regex:k_dec_scale|k_enc_prep' -s 2 -c 2 -o /tmp/prof_client -f python scripts/e2e_parts.py > gpurun_out/ncu_client.log 2>&1; echo "ncu rc=$?"
ncu -i /tmp/prof_client.ncu-rep --page raw --csv > gpurun_out/client_raw.csv 2>/dev/null
ncu -i /tmp/prof_client.ncu-rep --page source --csv --print-source sass -k regex:k_dec_scale > gpurun_out/client_src.csv 2>/dev/null
ls -la gpurun_out/client_*.csv
