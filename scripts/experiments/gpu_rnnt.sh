timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
timeout 900 python bench.py --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/bench4.json 2> gpurun_out/bench4.err; tail -3 gpurun_out/bench4.err
python -c "
import json; d=json.load(open('gpurun_out/bench4.json'))
print('value', d['value']/1e9, 'frac', d['roofline']['frac'], 'e2e', d['e2e']['value']/1e9)
print('rnnt', json.dumps(d['decode_rnnt']))
print('ctc', json.dumps(d['decode_ctc']))
"
