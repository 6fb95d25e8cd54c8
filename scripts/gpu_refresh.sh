#!/bin/bash
# Refresh every workload's numbers on the current build: default bench line (configs[1] +
# configs[2] sample), configs[4] ablation, configs[3] CIFAR (both schedules, 2-image sample).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python bench.py --steps 5 --warmup 3 > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; echo "bench rc=$?"
timeout 900 python bench.py --workload ablation --images 32 --steps 1 --warmup 1 > gpurun_out/ablation.json 2> gpurun_out/ablation.err; echo "ablation rc=$?"
for sched in hoisted reference; do
  timeout 1200 python bench.py --workload cifar --schedule $sched > gpurun_out/cifar_$sched.json 2> gpurun_out/cifar_$sched.err
  echo "cifar $sched rc=$?"
done
