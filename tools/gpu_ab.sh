set -x
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 900 python bench.py > gpurun_out/bench_now.json 2> gpurun_out/bench_now.err; tail -3 gpurun_out/bench_now.err
python -c "
import json; d=json.loads(open('gpurun_out/bench_now.json').read().strip().splitlines()[-1])
print('value', d['value'], d['unit'], 'frac', d['roofline']['frac'])
for k,v in d.get('per_m',{}).items(): print(k, v)
print('prefill', d.get('prefill'))
print('e2e', d.get('e2e'))
print('clocks', d.get('clocks'))
"
