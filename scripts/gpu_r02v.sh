# warp-local fences in the cluster cores (rings 2^15 / 2^16): parity + rotation rate at configs[3]'s parameters
python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "N16384 or N32768" > gpurun_out/t_big.log 2>&1; tail -2 gpurun_out/t_big.log
python scripts/bench_big_ring.py > gpurun_out/big_cur.json 2>gpurun_out/big_cur.err; cat gpurun_out/big_cur.json | head -c 1200; echo
FFCONV_HE_LIB=$PWD/build/var/libffconv_he_head.so python scripts/bench_big_ring.py > gpurun_out/big_head.json 2>gpurun_out/big_head.err; cat gpurun_out/big_head.json | head -c 1200; echo
