#!/bin/bash
# Compare library build variants (FFCONV_HE_LIB) on the GPU parity suite and the configs[1] rotation bench.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for lib in "" ${VARIANTS}; do
  tag=${lib:-default}; tag=$(basename "$tag" .so)
  echo "=== $tag"
  FFCONV_HE_LIB=$lib timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/var_$tag.pytest 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/var_$tag.pytest
  FFCONV_HE_LIB=$lib timeout 300 python bench.py --steps 5 --warmup 3 --no-inference > gpurun_out/var_$tag.json 2> gpurun_out/var_$tag.err; echo "bench rc=$?"
  python -c "import json; d=json.load(open('gpurun_out/var_$tag.json')); print(round(d['value']), {k: round(v['ms'],2) for k,v in d['kernels'].items()}, d['roofline']['frac'])"
done
