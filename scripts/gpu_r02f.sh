#!/bin/bash
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_stack.py -x -q -k "level_schedule or cfg0" 2>&1 | tail -3
for V in "" "FHE_KS_VARIANT=4" "FHE_KS_VARIANT=5"; do
  env $V timeout 300 python bench.py --steps 5 --warmup 3 --no-inference > gpurun_out/b.json 2> gpurun_out/b.err
  python - "$V" <<'PY'
import json, sys
d = json.loads(open("gpurun_out/b.json").read().strip().splitlines()[-1])
print(sys.argv[1] or "default", round(d["value"]), round(d["rates"]["rotation_frac_of_int_peak"], 3), {k: (v["calls"], round(v["ms"], 2)) for k, v in d["kernels"].items()})
PY
done
for LS in "" "--no-level-schedule"; do
  timeout 900 python bench.py --workload inference --images 64 --steps 1 --warmup 1 $LS > gpurun_out/inf.json 2> gpurun_out/inf.err
  python - "$LS" <<'PY'
import json, sys
d = json.loads(open("gpurun_out/inf.json").read().strip().splitlines()[-1])
i = d["inference"]
print(sys.argv[1] or "level-schedule", round(i["images_per_s"], 3), round(i["e2e_images_per_s"], 3), round(i["roofline"]["frac"], 3), i["logits_check"]["logits_match"])
PY
done
timeout 900 python bench.py --workload cifar --images 2 --chunk 2 > gpurun_out/cifar2.json 2> gpurun_out/cifar2.err; echo "cifar rc=$?"
python - <<'PY'
import json
d = json.loads(open("gpurun_out/cifar2.json").read().strip().splitlines()[-1])
c = d["cifar"]
print({k: c.get(k) for k in ("images_per_s", "ms", "wall_s", "logical_rotations", "logits_match_reference", "logits_match_oracle", "distinct_rotation_keys", "key_bytes_resident")})
PY
