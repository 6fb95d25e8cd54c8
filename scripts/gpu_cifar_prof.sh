#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
timeout 1500 python -m cProfile -o gpurun_out/cifar.prof bench.py --workload cifar > gpurun_out/cifar_cp.json 2> gpurun_out/cifar_cp.err; echo "cifar rc=$?"; tail -2 gpurun_out/cifar_cp.err
