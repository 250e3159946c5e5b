cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_advance_gpu.py -x -q > gpurun_out/adv_tests.log 2>&1; echo rc=$? >> gpurun_out/adv_tests.log
for env in "PGPB_ADVANCE_VARIANT=6" "PGPB_ADVANCE_VARIANT=8" "PGPB_ADVANCE_VARIANT=8 PGPB_V8_CTAS=1" "PGPB_ADVANCE_VARIANT=8 PGPB_V8_CTAS=3"; do
  echo "$env" >> gpurun_out/adv_pdl.log
  env $env timeout 300 python bench.py --no-decode --no-cpu-baseline 2>&1 | python -c "import json,sys; d=json.loads([l for l in sys.stdin if l.startswith('{')][0]); print(d['ms_per_step'], d['roofline']['frac'])" >> gpurun_out/adv_pdl.log
done
