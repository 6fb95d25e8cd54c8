#!/bin/bash
# key inner-product variants (FHE_KS_VARIANT) of a library build: parity, then the rotation bench
mkdir -p gpurun_out
[ -n "$LIB" ] && export FFCONV_HE_LIB=$PWD/$LIB
for v in ${KSV:-2 6 7 8}; do
  FHE_KS_VARIANT=$v python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "key_switch_stages or cfg1_full or rotate_many or rotate_multi or rotate_hoisted or composite or ops_bit_exact" > gpurun_out/ksv_$v.pytest 2>&1; rc=$?
  FHE_KS_VARIANT=$v python bench.py --steps 10 --warmup 3 --no-inference > gpurun_out/ksv_$v.json 2>gpurun_out/ksv_$v.err
  python -c "import json; d=json.load(open('gpurun_out/ksv_$v.json')); print('ksv=$v parity rc=$rc', round(d['value']), round(d['e2e']['value']), {k: round(v['ms'],2) for k,v in d['kernels'].items()})"
done
