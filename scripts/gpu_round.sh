#!/bin/bash
# One GPU session: tests, bench, launch list, one full ncu capture of the top kernel.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
python -m pytest tests -m gpu -x -q 2>&1 | tail -15
BENCH="python bench.py --steps 3 --warmup 3"
$BENCH > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
cat gpurun_out/bench.json
tail -5 gpurun_out/bench.err
if [ "${NCU:-1}" = "1" ]; then
  $BENCH > gpurun_out/plain.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -s 40 -c 400 --csv \
      --log-file gpurun_out/launches.csv $BENCH > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
  $BENCH > gpurun_out/plain2.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:${KERNEL:-k_modup} -s 3 -c 1 \
      -o gpurun_out/prof_top -f $BENCH > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?"
  tail -3 gpurun_out/ncu_full.log
fi
