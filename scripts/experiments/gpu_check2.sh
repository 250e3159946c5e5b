timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -15
timeout 600 python bench.py --steps 50 --warmup 5 > gpurun_out/bench2.json 2> gpurun_out/bench2.err; tail -3 gpurun_out/bench2.err
python -c "
import json; d=json.load(open('gpurun_out/bench2.json'))
print('value', d['value']/1e9, 'Gcells/s', 'roofline', d['roofline']['achieved'], d['roofline']['frac'])
print('e2e', d['e2e']['value']/1e9, 'clocks', d['clocks'])
print('decode', json.dumps(d['decode']))
print('cpu', d.get('cpu_baseline'))
"
