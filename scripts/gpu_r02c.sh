#!/bin/bash
set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -3
for V in "" "FHE_KS_BATCH=59" "FHE_KS_BATCH=29" "FHE_KS_FUSED=0"; do
  env $V timeout 300 python bench.py --steps 5 --warmup 3 --no-inference > gpurun_out/b.json 2> gpurun_out/b.err
  python - "$V" <<'PY'
import json, sys
d = json.loads(open("gpurun_out/b.json").read().strip().splitlines()[-1])
print(sys.argv[1] or "default", round(d["value"]), round(d["rates"]["rotation_frac_of_int_peak"], 3), {k: (v["calls"], round(v["ms"], 2)) for k, v in d["kernels"].items()})
PY
done
