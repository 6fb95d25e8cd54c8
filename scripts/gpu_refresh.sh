#!/bin/bash
# Refresh the secondary workloads on the current build: configs[4] ablation (64 images per GPU,
# every variant's logits checked) and configs[3] CIFAR (2-image sample, reference schedule).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1500 python bench.py --workload ablation --images 64 --steps 1 --warmup 1 > gpurun_out/ablation.json 2> gpurun_out/ablation.err; echo "ablation rc=$?"
timeout 1500 python bench.py --workload cifar --schedule reference > gpurun_out/cifar_reference.json 2> gpurun_out/cifar_reference.err; echo "cifar rc=$?"
head -c 600 gpurun_out/ablation.json; echo; head -c 600 gpurun_out/cifar_reference.json; echo
