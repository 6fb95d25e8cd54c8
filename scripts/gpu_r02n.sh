# pipelined key inner product (FHE_KS_VARIANT=4) against the default
python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "ops_bit_exact or composite" > gpurun_out/t_ks4.log 2>&1; tail -2 gpurun_out/t_ks4.log
FHE_KS_VARIANT=4 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "ops_bit_exact or composite" > gpurun_out/t_ks4b.log 2>&1; tail -2 gpurun_out/t_ks4b.log
run() {
  python bench.py --steps 5 --warmup 3 --no-inference > gpurun_out/$1.json 2>gpurun_out/$1.err
  python -c "
import json; d=json.load(open('gpurun_out/$1.json'))
print('$1', round(d['value']), {k: round(v['ms'],2) for k,v in d['kernels'].items()})"
}
run ksv2
FHE_KS_VARIANT=4 run ksv4
FHE_KS_VARIANT=4 FHE_KS_BATCH=128 run ksv4_s128
FHE_KS_BATCH=128 run ksv2_s128
