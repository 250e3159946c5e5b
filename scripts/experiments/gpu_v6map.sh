# advance v6: blocked vs strided row map (parity under both, bench sweep A/B)
cd $GRAFT_REPO_ROOT
PGPB_V6_MAP=1 timeout 900 python -m pytest tests/test_advance_gpu.py -x -q > gpurun_out/v6map_tests.log 2>&1; echo rc=$? >> gpurun_out/v6map_tests.log
for rep in 1 2; do for m in 0 1; do
  echo "== map $m"; PGPB_V6_MAP=$m timeout 300 python bench.py --no-decode --no-cpu-baseline 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('headline', round(d['roofline']['frac'],4), {k: round(v['frac_hbm'],4) for k,v in d['advance_sweep'].items() if isinstance(v,dict)})"
done; done > gpurun_out/v6map.log 2>&1
