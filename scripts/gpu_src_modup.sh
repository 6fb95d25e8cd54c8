#!/bin/bash
# SASS-level source page of one k_modup launch (stall samples and executed instructions per line)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
BENCH="python bench.py --steps 2 --warmup 3 --no-inference"
$BENCH > /dev/null 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:${KERNEL:-k_modup} -s 5 -c 1 -o /tmp/prof_src -f $BENCH > gpurun_out/ncu_src.log 2>&1; echo "ncu rc=$?"
ncu -i /tmp/prof_src.ncu-rep --page source --csv --print-source sass > gpurun_out/src_${KERNEL:-k_modup}.csv 2>/dev/null
ls -la gpurun_out/src_*.csv
