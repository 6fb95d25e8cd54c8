#!/bin/bash
# GPU regression check: full GPU parity suite, configs[1] rotation bench, NTT core rates at three prime sizes.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_gpu.log
timeout 300 python bench.py --steps 5 --warmup 3 --no-inference > gpurun_out/bench_rot.json 2> gpurun_out/bench_rot.err; echo "bench rc=$?"
python -c "import json; d=json.load(open('gpurun_out/bench_rot.json')); print(round(d['value']), round(d['e2e']['value']), {k: round(v['ms'],2) for k,v in d['kernels'].items()}, d['roofline']['frac'], d['roofline']['peaks_gmodmul'])"
for qb in 40 58 60; do QBITS=$qb WS=4,5 timeout 120 python scripts/ntt_bench.py > gpurun_out/ntt_q$qb.json 2>&1; echo "ntt q$qb rc=$?"; python -c "import json; d=json.load(open('gpurun_out/ntt_q$qb.json')); print({k:(round(v['us_per_row'],2), round(v['frac'],3), v['mismatch_rows']) for k,v in d.items() if isinstance(v, dict)})"; done
