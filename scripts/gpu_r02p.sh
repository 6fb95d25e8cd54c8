# parity + bench of the current build and variants
python -m pytest tests/test_gpu_parity.py tests/test_gpu_variants.py -m gpu -x -q > gpurun_out/t_keep.log 2>&1; tail -3 gpurun_out/t_keep.log
run() {
  python bench.py --steps 5 --warmup 3 --no-inference > gpurun_out/$1.json 2>gpurun_out/$1.err
  python -c "
import json; d=json.load(open('gpurun_out/$1.json'))
print('$1', round(d['value']), 'e2e', round(d['e2e']['value']), {k: round(v['ms'],2) for k,v in d['kernels'].items()}, round(d['rates']['rescale_per_s']))"
}
run cur
for v in $VARIANTS; do
FFCONV_HE_LIB=$PWD/build/var/libffconv_he_$v.so run $v
done
