#!/bin/bash
# ncu --set full of one kernel inside the rotation bench: KERNEL=<regex> TAG=<name>
set -x
mkdir -p gpurun_out
BENCH="python bench.py --steps 2 --warmup 3 --no-inference"
$BENCH > gpurun_out/plain_$TAG.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:$KERNEL -s ${SKIP:-5} -c 1 \
    -o gpurun_out/prof_$TAG -f $BENCH > gpurun_out/ncu_$TAG.log 2>&1; echo "ncu $TAG rc=$?"
tail -3 gpurun_out/ncu_$TAG.log
