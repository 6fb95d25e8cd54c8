#!/bin/bash
# ring 2^16 (configs[3] parameters): rotation rate, per-kernel times, and full ncu captures of the
# cluster-row ModUp and ModDown kernels (active clusters, occupancy, pipe busy)
mkdir -p gpurun_out
python scripts/bench_big_ring.py > gpurun_out/big_ring.json 2> gpurun_out/big_ring.err; echo "rc=$?"; cat gpurun_out/big_ring.json
for K in k_modup k_rescale; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -s 2 -c 1 -o /tmp/prof_big_$K -f python scripts/bench_big_ring.py > gpurun_out/ncu_big_$K.log 2>&1; echo "ncu $K rc=$?"
  python scripts/ncu_digest.py /tmp/prof_big_$K.ncu-rep gpurun_out/r02_ring16_${K#k_}.txt 30
done
grep -n "Cluster\|Waves Per SM\|Grid Size\|Achieved Occ\|fmaheavy\|Duration" gpurun_out/r02_ring16_modup.txt gpurun_out/r02_ring16_rescale.txt | head -40
