# advance kernel: parity tests, then bench ms/step and roofline fraction (HEAD lib vs working tree, twice)
cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_advance_gpu.py -x -q > gpurun_out/adv_tests.log 2>&1; echo rc=$? >> gpurun_out/adv_tests.log
: > gpurun_out/adv_exp.log
for i in 1 2; do
for lib in paper_2508_07014_b200/build/libpgpb_head.so paper_2508_07014_b200/libpgpb.so; do
  echo "$lib" >> gpurun_out/adv_exp.log
  PGPB_LIB_PATH=$lib timeout 300 python bench.py --no-decode --no-cpu-baseline 2>&1 | python -c "import json,sys; d=json.loads([l for l in sys.stdin if l.startswith('{')][0]); print(d['ms_per_step'], d['roofline']['frac'])" >> gpurun_out/adv_exp.log
done
done
