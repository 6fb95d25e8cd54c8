#!/bin/bash
# NTT core variants (old W4/W5 vs two-phase E16/E32) and key-switching sub-batch sizes
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
WS=4,5,200,201 timeout 300 python scripts/ntt_bench.py 1184 > gpurun_out/ntt_wp.json 2> gpurun_out/ntt_wp.err; echo "ntt rc=$?"
for S in 64 74 80; do
  FHE_KS_BATCH=$S timeout 300 python bench.py --steps 3 --warmup 3 --no-inference > gpurun_out/ksb$S.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/ksb$S.json')); print($S, round(d['value']), {k: round(v['ms'],2) for k,v in d['kernels'].items()})"
done
