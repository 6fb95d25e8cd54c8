#!/bin/bash
set -x
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q --durations=12 2>&1 | tail -22
timeout 900 python bench.py --workload cifar --images 64 --chunk 64 > gpurun_out/cifar64.json 2> gpurun_out/cifar64.err; echo "cifar rc=$?"
tail -2 gpurun_out/cifar64.err
python - <<'PY'
import json
d = json.loads(open("gpurun_out/cifar64.json").read().strip().splitlines()[-1])
c = d["cifar"]
print({k: c[k] for k in ("images_per_s", "ms", "wall_s", "logical_rotations", "logits_checked", "logits_match_reference", "key_bytes_resident", "L", "crt_primes", "gpu_launches")})
PY
