for v in 0 1 2 3; do
  FHE_KS_VARIANT=$v python bench.py --steps 3 --warmup 3 --no-inference > gpurun_out/ksv$v.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/ksv$v.json')); print($v, round(d['value']), d['kernels']['k_ks_inner']['ms'])"
done
