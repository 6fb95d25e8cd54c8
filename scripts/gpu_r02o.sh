# e2e pipeline modes and chunk counts (rotation microbench), default sub-batch 128
run() {
  python bench.py --steps 5 --warmup 3 --no-inference > gpurun_out/$1.json 2>gpurun_out/$1.err
  python -c "
import json; d=json.load(open('gpurun_out/$1.json'))
print('$1', round(d['value']), 'e2e', round(d['e2e']['value']), d['e2e']['check'])"
}
BENCH_E2E_MODE=phases run e2e_phases8
BENCH_E2E_MODE=pipeline BENCH_E2E_CHUNKS=8 run e2e_pipe8
BENCH_E2E_MODE=pipeline BENCH_E2E_CHUNKS=4 run e2e_pipe4
BENCH_E2E_MODE=pipeline BENCH_E2E_CHUNKS=16 run e2e_pipe16
BENCH_E2E_MODE=pipeline BENCH_E2E_CHUNKS=2 run e2e_pipe2
