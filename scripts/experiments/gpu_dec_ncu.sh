timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
echo "B=128 $(timeout 300 python scripts/decode_sweep.py 128)"
echo "B=1024 $(timeout 300 python scripts/decode_sweep.py 1024)"
ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none --csv --log-file gpurun_out/dec_launches.csv python scripts/prof_kernels.py greedy 2 > /dev/null 2>&1
python - <<'PY'
import csv
rows=[r for r in csv.reader(open('gpurun_out/dec_launches.csv')) if len(r)>10]
hdr=rows[0]
for r in rows[1:]:
    d=dict(zip(hdr,r))
    if 'pgpb' in d['Kernel Name']: print(d['Kernel Name'][:45], d['Metric Name'], d['Metric Value'])
PY
