# advance v6 with the table's ranked bitmap rows (A/B vs the per-row build), parity first
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_advance_gpu.py tests/test_shim_gpu.py -x -q > gpurun_out/tbits_tests.log 2>&1; echo rc=$? >> gpurun_out/tbits_tests.log
PGPB_V6_MAP=1 timeout 900 python -m pytest tests/test_advance_gpu.py -x -q >> gpurun_out/tbits_tests.log 2>&1; echo rc=$? >> gpurun_out/tbits_tests.log
for rep in 1 2; do for tb in 0 1; do
  echo "== tbits $tb"; PGPB_V6_TBITS=$tb timeout 300 python bench.py --no-decode --no-cpu-baseline 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('headline', round(d['roofline']['frac'],4), {k: round(v['frac_hbm'],4) for k,v in d['advance_sweep'].items() if isinstance(v,dict)})"
done; done > gpurun_out/tbits.log 2>&1
