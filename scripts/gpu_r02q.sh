#!/bin/bash
# round-2 final evidence: launch list of the rotation bench + full captures of the key-switch kernels
mkdir -p gpurun_out
BENCH="python bench.py --steps 2 --warmup 3 --no-inference"
$BENCH > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -s 100 -c 500 --csv \
    --log-file gpurun_out/launches_${TAG:-r02b}.csv $BENCH > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
for K in ${KERNELS:-k_modup k_rescale}; do
  ncu --set full --clock-control none --import-source on -k regex:$K -s 5 -c 1 \
      -o /tmp/prof_$K -f $BENCH > gpurun_out/ncu_full_$K.log 2>&1; echo "ncu $K rc=$?"
  python scripts/ncu_digest.py /tmp/prof_$K.ncu-rep gpurun_out/digest_${TAG:-r02b}_$K.txt 40
done
python scripts/summarize_ncu.py gpurun_out/launches_${TAG:-r02b}.csv > gpurun_out/launches_${TAG:-r02b}.txt 2>&1
ls -la gpurun_out | tail -8
