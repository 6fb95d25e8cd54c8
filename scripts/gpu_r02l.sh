# composite operators (fhe_rotate_and_sum / fhe_combine / fhe_ct_gemm) parity, whole GPU suite,
# and the L1 cache-policy variants of the row kernels
python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "composite or ct_gemm" > gpurun_out/t_comp.log 2>&1; tail -5 gpurun_out/t_comp.log
python -m pytest tests -m gpu -x -q > gpurun_out/gputest.log 2>&1; tail -3 gpurun_out/gputest.log
python bench.py --steps 5 --warmup 3 --no-inference > gpurun_out/base.json 2>/dev/null
python -c "
import json; d=json.load(open('gpurun_out/base.json'))
print('base', round(d['value']), {k: round(v['ms'],2) for k,v in d['kernels'].items()})"
for v in l1p l1p9; do
  FFCONV_HE_LIB=$PWD/build/var/libffconv_he_$v.so python bench.py --steps 5 --warmup 3 --no-inference > gpurun_out/$v.json 2>gpurun_out/$v.err
  python -c "
import json; d=json.load(open('gpurun_out/$v.json'))
print('$v', round(d['value']), {k: round(v['ms'],2) for k,v in d['kernels'].items()})"
done
