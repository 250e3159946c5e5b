timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -4
timeout 600 python bench.py --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/bench3.json 2> gpurun_out/bench3.err; tail -3 gpurun_out/bench3.err
python -c "
import json; d=json.load(open('gpurun_out/bench3.json'))
print('value', d['value']/1e9, 'Gcells/s', 'roofline', d['roofline']['achieved'], d['roofline']['frac'])
print('e2e', d['e2e']['value']/1e9, 'clocks', d['clocks'])
print('decode', json.dumps(d['decode']))
"
