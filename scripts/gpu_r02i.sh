#!/bin/bash
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_variants.py tests/test_gpu_stack.py -x -q -k "variant or captured or level_schedule" 2>&1 | tail -3
timeout 600 python bench.py --workload latency --steps 1 --warmup 1 > gpurun_out/latency.json 2> gpurun_out/latency.err; echo "latency rc=$?"
cat gpurun_out/latency.json; tail -3 gpurun_out/latency.err
for V in "FHE_KS_BATCH=74" "FHE_KS_BATCH=96"; do
  env $V timeout 300 python bench.py --steps 5 --warmup 3 --no-inference > gpurun_out/b.json 2> gpurun_out/b.err
  python - "$V" <<'PY'
import json, sys
d = json.loads(open("gpurun_out/b.json").read().strip().splitlines()[-1])
print(sys.argv[1], round(d["value"]), round(d["rates"]["rotation_frac_of_int_peak"], 3), {k: (v["calls"], round(v["ms"], 2)) for k, v in d["kernels"].items()})
PY
done
for V in "FHE_KS_FUSED=0" "FHE_KS_FUSED=1"; do
  env $V timeout 900 python bench.py --workload inference --images 64 --steps 1 --warmup 1 > gpurun_out/inf.json 2> gpurun_out/inf.err
  python - "$V" <<'PY'
import json, sys
d = json.loads(open("gpurun_out/inf.json").read().strip().splitlines()[-1])
i = d["inference"]
print(sys.argv[1], round(i["images_per_s"], 3), round(i["roofline"]["frac"], 3), i["logits_check"]["logits_match"], {k: v["ms"] for k, v in i["kernel_ms_one_chunk"].items() if v["ms"] > 50})
PY
  env $V timeout 900 python bench.py --workload cifar --images 2 --chunk 2 > gpurun_out/cifar.json 2> gpurun_out/cifar.err
  python - "$V" <<'PY'
import json, sys
d = json.loads(open("gpurun_out/cifar.json").read().strip().splitlines()[-1])
c = d["cifar"]
print(sys.argv[1], "cifar", {k: c.get(k) for k in ("images_per_s", "ms", "logits_match_reference", "logits_match_oracle")})
PY
done
FHE_BENCH_PROF=1 timeout 900 python bench.py --workload cifar --images 2 --chunk 2 > gpurun_out/cifar_prof.json 2> gpurun_out/cifar_prof.err
python - <<'PY'
import json
d = json.loads(open("gpurun_out/cifar_prof.json").read().strip().splitlines()[-1])
print("cifar prof", {k: v for k, v in d["cifar"]["kernel_ms"].items() if v["ms"] > 200})
PY
