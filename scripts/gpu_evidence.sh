#!/bin/bash
# round-2 final evidence: launch list of the rotation bench, full captures of the five key-switch
# kernels, the ct-GEMM and the hoisted GEMM, digested on the box (scripts/ncu_digest.py)
mkdir -p gpurun_out
BENCH="python bench.py --steps 2 --warmup 3 --no-inference"
$BENCH > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -s 100 -c 500 --csv \
    --log-file gpurun_out/launches_r02final.csv $BENCH > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
python scripts/summarize_ncu.py gpurun_out/launches_r02final.csv gpurun_out/r02_rotation
for K in k_modup k_rescale k_rot_gather_intt k_ks_special k_ks_inner; do
  ncu --set full --clock-control none --import-source on -k regex:$K -s 5 -c 1 \
      -o /tmp/prof_$K -f $BENCH > gpurun_out/ncu_full_$K.log 2>&1; echo "ncu $K rc=$?"
  python scripts/ncu_digest.py /tmp/prof_$K.ncu-rep gpurun_out/r02_$K.txt 40
done
# hoisted GEMM and ct-GEMM: a small inference sample / the composite-operator test
INF="python bench.py --workload inference --images 64 --steps 1 --warmup 0 --schedule hoisted"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_hoisted_dot -s 2 -c 1 \
    -o /tmp/prof_hoist -f $INF > gpurun_out/ncu_full_hoist.log 2>&1; echo "ncu hoist rc=$?"
python scripts/ncu_digest.py /tmp/prof_hoist.ncu-rep gpurun_out/r02_k_hoisted_dot.txt 30
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_ct_gemm -c 1 \
    -o /tmp/prof_gemm -f python scripts/ct_gemm_probe.py > gpurun_out/ncu_full_gemm.log 2>&1; echo "ncu gemm rc=$?"
python scripts/ncu_digest.py /tmp/prof_gemm.ncu-rep gpurun_out/r02_k_ct_gemm.txt 30
python scripts/ct_gemm_probe.py > gpurun_out/r02_ct_gemm.json 2>gpurun_out/ct_gemm.err; cat gpurun_out/r02_ct_gemm.json
ls -la gpurun_out | tail -12
