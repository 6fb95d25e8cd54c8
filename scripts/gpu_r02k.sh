# cluster rows (2 CTAs x 2^13 words) at ring 2^14: two CTAs per SM overlap each other's barriers
export FFCONV_HE_LIB=$PWD/build/var/libffconv_he_l13.so
python -m pytest tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/t_l13.log 2>&1; tail -3 gpurun_out/t_l13.log
python bench.py --steps 5 --warmup 3 --no-inference > gpurun_out/l13.json 2>gpurun_out/l13.err
python -c "
import json; d=json.load(open('gpurun_out/l13.json'))
print('l13', round(d['value']), {k: round(v['ms'],2) for k,v in d['kernels'].items()})"
unset FFCONV_HE_LIB
python bench.py --workload latency > gpurun_out/latency.json 2>gpurun_out/latency.err; tail -c 1500 gpurun_out/latency.json
