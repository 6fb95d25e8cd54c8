#!/bin/bash
# round 2, session A: baseline tests, sanitizers on small rings, ncu of the modmul peak probe
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
for W in small ring14 cluster; do
  timeout 600 compute-sanitizer --tool memcheck --leak-check no python scripts/sanitize_smoke.py $W > gpurun_out/san_memcheck_$W.log 2>&1; echo "memcheck $W rc=$?"
done
for W in small cluster; do
  timeout 900 compute-sanitizer --tool racecheck --racecheck-report all python scripts/sanitize_smoke.py $W > gpurun_out/san_racecheck_$W.log 2>&1; echo "racecheck $W rc=$?"
  timeout 900 compute-sanitizer --tool synccheck python scripts/sanitize_smoke.py $W > gpurun_out/san_synccheck_$W.log 2>&1; echo "synccheck $W rc=$?"
done
python scripts/peak_probe.py > gpurun_out/peak_plain.log 2>&1 && \
ncu --set full --clock-control none -k regex:k_peak_modmul -c 4 -o gpurun_out/prof_peak -f python scripts/peak_probe.py > gpurun_out/ncu_peak.log 2>&1; echo "ncu peak rc=$?"
cat gpurun_out/peak_plain.log
tail -3 gpurun_out/san_*.log
