# rotate-and-add addend in the ModDown epilogue (default) vs folded into the inner product
python -m pytest tests/test_gpu_parity.py tests/test_gpu_variants.py -m gpu -x -q > gpurun_out/t_keep.log 2>&1; tail -2 gpurun_out/t_keep.log
for f in 0 1; do
FHE_FOLD_ACC=$f python bench.py --workload inference --images 64 --steps 1 --warmup 0 > gpurun_out/inf_fold$f.json 2>gpurun_out/inf_fold$f.err
python -c "
import json; d=json.loads(open('gpurun_out/inf_fold$f.json').read().strip().splitlines()[-1])
i=d.get('inference', d); print('fold_acc=$f', i.get('images_per_s'), i.get('logits_check',{}).get('logits_match'), {k: round(v['ms']) for k,v in i.get('kernel_ms_one_chunk',{}).items() if v['ms']>500})"
done
