# full GPU suite + default bench (rotation, configs[2] both schedules, configs[0] latency) + reference arm
python -m pytest tests -m gpu -x -q > gpurun_out/gputest.log 2>&1; tail -3 gpurun_out/gputest.log
python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; tail -c 300 gpurun_out/bench_default.err
python bench.py --impl reference > gpurun_out/bench_ref.json 2>gpurun_out/bench_ref.err
python -c "
import json; d=json.loads(open('gpurun_out/bench_default.json').read().strip().splitlines()[-1])
print(round(d['value']), round(d['e2e']['value']), d['roofline']['frac'], d['rates'])
print({k:(d[k]['images_per_s'], d[k]['roofline']['frac'], d[k]['logits_check']['logits_match']) for k in ('inference','inference_hoisted')})
print(d.get('latency_cfg0'))"
