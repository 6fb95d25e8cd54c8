#!/bin/bash
# A/B: library variants (VARIANTS="build/var/libffconv_he_x.so ...") against the in-tree build:
# the key-switch parity tests, then the configs[1] rotation bench of each.
mkdir -p gpurun_out
for lib in "" ${VARIANTS}; do
  tag=${lib:-default}; tag=$(basename "$tag" .so); tag=${tag#libffconv_he_}
  [ -n "$lib" ] && lib=$PWD/$lib
  FFCONV_HE_LIB=$lib python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "key_switch_stages or cfg1_full or rotate_many or rotate_hoisted" > gpurun_out/ab_$tag.pytest 2>&1; rc=$?
  FFCONV_HE_LIB=$lib python bench.py --steps 10 --warmup 3 --no-inference > gpurun_out/ab_$tag.json 2>gpurun_out/ab_$tag.err
  python -c "import json; d=json.load(open('gpurun_out/ab_$tag.json')); print('$tag', 'parity rc=$rc', round(d['value']), round(d['e2e']['value']), {k: round(v['ms'],2) for k,v in d['kernels'].items()}, round(d['roofline']['frac'],4))"
done
