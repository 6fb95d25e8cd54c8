#!/bin/bash
# ncu evidence for the current build: launch list + one full capture of the top kernel.
set -x
mkdir -p gpurun_out
BENCH="python bench.py --steps 2 --warmup 3 --no-inference"
$BENCH > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -s 100 -c 500 --csv \
    --log-file gpurun_out/launches.csv $BENCH > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
$BENCH > gpurun_out/plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:${KERNEL:-k_modup} -s 5 -c 1 \
    -o gpurun_out/prof_top -f $BENCH > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?"
$BENCH > gpurun_out/plain3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_ks_inner -s 5 -c 1 \
    -o gpurun_out/prof_ks -f $BENCH > gpurun_out/ncu_full2.log 2>&1; echo "ncu full2 rc=$?"
