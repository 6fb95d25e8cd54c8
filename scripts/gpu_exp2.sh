#!/bin/bash
# NTT forward experiments: L1-resident twiddles / no barriers (timing only), then an
# ncu source-level capture of the production forward core.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
WS=4,301,302,303 timeout 300 python scripts/ntt_bench.py 1184 > gpurun_out/ntt_exp.json 2> gpurun_out/ntt_exp.err; echo "ntt rc=$?"
WS=4 timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_bench_fwd -c 1 -f -o gpurun_out/ntt_fwd python scripts/ntt_bench.py 148 > gpurun_out/ncu_ntt.log 2>&1; echo "ncu rc=$?"
ls -la gpurun_out/
