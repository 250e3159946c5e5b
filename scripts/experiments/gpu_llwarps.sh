# label-loop step: warps per CTA A/B (RNN-T config 2 bench line)
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_rnnt_gpu.py -x -q > gpurun_out/ll_tests.log 2>&1; echo rc=$? >> gpurun_out/ll_tests.log
for rep in 1 2; do for w in 8 4 2 1; do
  echo "== warps $w"; PGPB_LL_WARPS=$w timeout 300 python bench.py --no-cpu-baseline 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['decode_rnnt']; print(round(r['unboosted']['ms'],3), round(r['boosted']['ms'],3), round(r['overhead'],4))"
done; done > gpurun_out/llwarps.log 2>&1
