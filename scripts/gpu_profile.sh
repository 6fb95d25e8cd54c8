#!/bin/bash
# ncu evidence for the current build: launch list + full captures of the top rotation kernels,
# summarised on the box (scripts/summarize_ncu.py) so only text comes back.
set -x
mkdir -p gpurun_out
BENCH="python bench.py --steps 2 --warmup 3 --no-inference"
$BENCH > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -s 100 -c 500 --csv \
    --log-file gpurun_out/launches.csv $BENCH > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
for K in ${KERNELS:-k_modup k_ks_inner k_rescale k_rot_gather_intt k_ks_special}; do
  $BENCH > gpurun_out/plain_$K.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:$K -s 5 -c 1 \
      -o /tmp/prof_$K -f $BENCH > gpurun_out/ncu_full_$K.log 2>&1; echo "ncu $K rc=$?"
done
python scripts/summarize_ncu.py gpurun_out/launches.csv gpurun_out/${TAG:-r01_rotation} /tmp/prof_*.ncu-rep > /dev/null
ls -la gpurun_out
