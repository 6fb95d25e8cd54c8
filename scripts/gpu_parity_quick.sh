#!/bin/bash
# GPU parity suite + a short rotation bench (regression check)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/pytest_gpu.log
timeout 300 python bench.py --steps 3 --warmup 3 --no-inference > gpurun_out/bench_rot.json 2> gpurun_out/bench_rot.err; echo "bench rc=$?"
python -c "import json; d=json.load(open('gpurun_out/bench_rot.json')); print(round(d['value']), d['rates'])"
