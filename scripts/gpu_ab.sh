#!/bin/bash
# A/B: the in-tree library against build/var/libffconv_he_head.so (parity first, then the rotation bench of both)
mkdir -p gpurun_out
python -m pytest tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/ab_parity.log 2>&1; echo "parity rc=$?"; tail -2 gpurun_out/ab_parity.log
for tag in new head new head; do
  lib=""; [ $tag = head ] && lib=$PWD/build/var/libffconv_he_head.so
  FFCONV_HE_LIB=$lib python bench.py --steps 10 --warmup 3 --no-inference > gpurun_out/ab_$tag.json 2>gpurun_out/ab_$tag.err
  python -c "import json; d=json.load(open('gpurun_out/ab_$tag.json')); print('$tag', round(d['value']), round(d['e2e']['value']), {k: round(v['ms'],2) for k,v in d['kernels'].items()}, round(d['roofline']['frac'],4), round(d['roofline']['peak'],1))"
done
