#!/bin/bash
# GPU parity suite, then configs[3] (CIFAR-shaped FFConv HECNN, ring 2^16) on a 2-image
# sample with logits checked against the reference fixture
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
for sched in reference; do
  timeout 1500 python bench.py --workload cifar --schedule $sched > gpurun_out/cifar_$sched.json 2> gpurun_out/cifar_$sched.err
  echo "$sched rc=$?"
  python -c "import json; d=json.load(open('gpurun_out/cifar_$sched.json')); c=d['cifar']; print({k: c[k] for k in ('images_per_s','ms','wall_s','logical_rotations','physical_rotations_per_s','logits_match_reference','key_bytes_resident','L','crt_primes')})" 2>&1 | tail -2
  tail -3 gpurun_out/cifar_$sched.err
done
