# multiplication-free centered lift + L1 policy default: parity, then rotation bench of the variants
python -m pytest tests/test_gpu_parity.py tests/test_gpu_variants.py -m gpu -x -q > gpurun_out/t_par.log 2>&1; tail -3 gpurun_out/t_par.log
run() {
  python bench.py --steps 5 --warmup 3 --no-inference > gpurun_out/$1.json 2>gpurun_out/$1.err
  python -c "
import json; d=json.load(open('gpurun_out/$1.json'))
print('$1', round(d['value']), {k: round(v['ms'],2) for k,v in d['kernels'].items()})"
}
run main
FFCONV_HE_LIB=$PWD/build/var/libffconv_he_nol1.so run nol1
FFCONV_HE_LIB=$PWD/build/var/libffconv_he_k13.so run k13
