#!/bin/bash
# ncu --set full (with source) of the rotation's key-switch kernels on the current build,
# digested on the box (scripts/ncu_digest.py) -- the reports are tens of MB each
set -x
mkdir -p gpurun_out
BENCH="python bench.py --steps 2 --warmup 3 --no-inference"
$BENCH > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -s 100 -c 500 --csv \
    --log-file gpurun_out/launches_${TAG:-r02}.csv $BENCH > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
for K in ${KERNELS:-k_rescale k_rot_gather_intt k_ks_special k_modup k_ks_inner}; do
  ncu --set full --clock-control none --import-source on -k regex:$K -s 5 -c 1 \
      -o /tmp/prof_$K -f $BENCH > gpurun_out/ncu_full_$K.log 2>&1; echo "ncu $K rc=$?"
  python scripts/ncu_digest.py /tmp/prof_$K.ncu-rep gpurun_out/digest_${TAG:-r02}_$K.txt 80
done
ls -la gpurun_out
