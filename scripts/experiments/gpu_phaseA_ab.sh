# phase-A reductions: insertion chains vs redux.sync (CREDUX) groups
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_ctc_fused_gpu.py tests/test_greedy_gpu.py tests/test_shim_gpu.py -x -q > gpurun_out/rx_tests.log 2>&1; echo rc=$? >> gpurun_out/rx_tests.log
export PGPB_REGIMES=clean,dense PGPB_IMPLS=fused
for rep in 1 2; do
for lib in chains rx; do
  for knob in "X=1" "PGPB_CTC_ONLY_A=1"; do
    echo "== $lib $knob"
    env $knob PGPB_LIB_PATH=paper_2508_07014_b200/build/libpgpb_$lib.so timeout 120 python scripts/ctc_regimes.py 2>&1 | tail -2
  done
done
done
