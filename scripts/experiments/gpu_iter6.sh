# full GPU suite + CTC regimes + walker stage costs
cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/gpu_tests.log
export PGPB_REGIMES=clean PGPB_IMPLS=fused
for knob in "PGPB_CTC_ONLY_A=1" "PGPB_CTC_STOP=1" "PGPB_CTC_STOP=2" "PGPB_CTC_STOP=3" "PGPB_CTC_STOP=4" "PGPB_CTC_STOP=5" "PGPB_CTC_STOP=6" "PGPB_CTC_STOP=7" "X=1"; do
  echo "== $knob"; env $knob timeout 120 python scripts/ctc_regimes.py 2>&1 | tail -1
done > gpurun_out/stops.log 2>&1
