# sub-batch sweep (wave quantization of the row kernels) + the captured-plan test
python -m pytest tests/test_gpu_stack.py -m gpu -x -q -k captured > gpurun_out/t_captured.log 2>&1; tail -3 gpurun_out/t_captured.log
for s in 37 64 74 111 128; do
  FHE_KS_BATCH=$s python bench.py --steps 5 --warmup 3 --no-inference > gpurun_out/ksb$s.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/ksb$s.json'))
print($s, round(d['value']), {k: round(v['ms'],2) for k,v in d['kernels'].items()})"
done
for ln in 1 3; do
  FHE_LANES=$ln FHE_KS_BATCH=74 python bench.py --steps 5 --warmup 3 --no-inference > gpurun_out/ksb74_l$ln.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/ksb74_l$ln.json'))
print('lanes', $ln, round(d['value']))"
done
