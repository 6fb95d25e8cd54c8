#!/bin/bash
# round 2, session B: fused key switching (TMEM) parity + first rotation numbers
set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -15
timeout 300 python bench.py --steps 5 --warmup 3 --no-inference > gpurun_out/b_fused.json 2> gpurun_out/b_fused.err; echo "bench fused rc=$?"
FHE_KS_FUSED=0 timeout 300 python bench.py --steps 5 --warmup 3 --no-inference > gpurun_out/b_unfused.json 2> gpurun_out/b_unfused.err; echo "bench unfused rc=$?"
python - <<'PY'
import json
for f in ("gpurun_out/b_fused.json", "gpurun_out/b_unfused.json"):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        print(f, round(d["value"]), d["rates"]["rotation_frac_of_int_peak"], {k: (v["calls"], round(v["ms"], 2)) for k, v in d["kernels"].items()}, d["e2e"]["check"])
    except Exception as e:
        print(f, "ERR", e, open(f.replace(".json", ".err")).read()[-2000:])
PY
