#!/bin/bash
# configs[2] chunk-size sweep (images per plan walk) and lane count
mkdir -p gpurun_out
for c in 128 256; do
  timeout 900 python bench.py --workload inference --images 256 --chunk $c --steps 1 --warmup 1 > gpurun_out/inf_chunk$c.json 2> gpurun_out/inf_chunk$c.err; echo "chunk $c rc=$?"
  python - <<P
import json
try:
    d=json.load(open('gpurun_out/inf_chunk$c.json')); i=d['inference']; print($c, i['images_per_s'], i['e2e_images_per_s'], i['roofline']['frac'], i['logits_check']['logits_match'], i['gpu_launches'])
except Exception as e: print('fail', e)
P
  tail -2 gpurun_out/inf_chunk$c.err
done
FHE_LANES=3 timeout 900 python bench.py --workload inference --images 256 --chunk 64 --steps 1 --warmup 1 > gpurun_out/inf_lanes3.json 2> gpurun_out/inf_lanes3.err
python - <<P
import json
d=json.load(open('gpurun_out/inf_lanes3.json')); i=d['inference']; print('lanes3', i['images_per_s'], i['roofline']['frac'], i['logits_check']['logits_match'])
P
FHE_LANES=3 python bench.py --no-inference > gpurun_out/rot_lanes3.json 2>/dev/null
python - <<P
import json
d=json.load(open('gpurun_out/rot_lanes3.json')); print('rot lanes3', d['value'], d['e2e']['value'])
P
