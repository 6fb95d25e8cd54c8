#!/bin/bash
# ncu --set full of the three NTT-bearing rotation kernels (one launch each) after a clean bench run.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
BENCH="python bench.py --steps 2 --warmup 3 --no-inference"
$BENCH > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k 'regex:k_modup|k_rescale|k_rot_gather' -s 30 -c 3 \
    -o gpurun_out/prof3 -f $BENCH > gpurun_out/ncu_prof3.log 2>&1; echo "ncu rc=$?"
tail -2 gpurun_out/ncu_prof3.log
