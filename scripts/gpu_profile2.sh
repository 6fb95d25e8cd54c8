#!/bin/bash
set -x
mkdir -p gpurun_out
BENCH="python bench.py --steps 2 --warmup 3 --no-inference"
$BENCH > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_rescale -s 5 -c 1 \
    -o /tmp/prof_rescale -f $BENCH > gpurun_out/ncu_r.log 2>&1; echo "ncu rescale rc=$?"
$BENCH > gpurun_out/plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_rot_gather -s 5 -c 1 \
    -o /tmp/prof_gather -f $BENCH > gpurun_out/ncu_g.log 2>&1; echo "ncu gather rc=$?"
INF="python bench.py --workload inference --images 8 --chunk 8 --steps 1 --warmup 1 --schedule hoisted"
$INF > gpurun_out/plain3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_hoisted_dot -s 2 -c 1 \
    -o gpurun_out/prof_hoist -f $INF > gpurun_out/ncu_h.log 2>&1; echo "ncu hoist rc=$?"
python scripts/summarize_ncu.py /dev/null gpurun_out/r01 /tmp/prof_rescale.ncu-rep /tmp/prof_gather.ncu-rep gpurun_out/prof_hoist.ncu-rep > gpurun_out/summ.log 2>&1
ls -la gpurun_out
