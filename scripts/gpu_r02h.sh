#!/bin/bash
# configs[3] at its stated 64 images (chunks of 16), every image's logits checked; then the
# configs[4] ablation on 64 images per variant with logits checked
set -x
mkdir -p gpurun_out
timeout 600 python bench.py --workload ablation --images 64 --chunk 64 > gpurun_out/ablation_r02.json 2> gpurun_out/ablation_r02.err; echo "ablation rc=$?"
timeout 6000 python bench.py --workload cifar --images 64 --chunk 16 > gpurun_out/cifar64_r02.json 2> gpurun_out/cifar64_r02.err; echo "cifar rc=$?"
tail -3 gpurun_out/cifar64_r02.err
