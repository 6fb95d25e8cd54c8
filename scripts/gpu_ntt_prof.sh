#!/bin/bash
# ncu --set full of the standalone forward and inverse NTT cores (radix-16, n = 2^14, 40-bit q)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
QBITS=40 WS=4 python scripts/ntt_bench.py > /dev/null 2>&1 && \
QBITS=40 WS=4 timeout 600 ncu --set full --clock-control none --import-source on -k 'regex:k_bench_inv' -s 3 -c 1 \
    -o /tmp/prof_ntt -f python scripts/ntt_bench.py > gpurun_out/ncu_ntt.log 2>&1; echo "ncu rc=$?"
ncu -i /tmp/prof_ntt.ncu-rep --page raw --csv > gpurun_out/ntt_raw.csv 2>/dev/null
ncu -i /tmp/prof_ntt.ncu-rep --page source --csv --print-source sass -k regex:k_bench_inv > gpurun_out/ntt_inv_src.csv 2>/dev/null
ls -la gpurun_out/ntt_raw.csv gpurun_out/ntt_inv_src.csv
