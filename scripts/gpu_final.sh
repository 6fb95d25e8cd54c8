#!/bin/bash
# Round-end validation on one B200: GPU tests, smoke(), the default bench line and the reference arm.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
( time python -m pytest tests -m gpu -x -q ) > gpurun_out/final_tests.log 2>&1; echo "tests rc=$?"; tail -4 gpurun_out/final_tests.log
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/final_smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/final_smoke.log
( time python bench.py ) > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err; echo "bench rc=$?"
head -c 1500 gpurun_out/final_bench.json; echo; tail -4 gpurun_out/final_bench.err
( time python bench.py --impl reference ) > gpurun_out/final_bench_ref.json 2> gpurun_out/final_bench_ref.err; echo "ref rc=$?"
head -c 800 gpurun_out/final_bench_ref.json; echo; tail -4 gpurun_out/final_bench_ref.err
