# walker: L1 prefetch of the first closure entries (A/B), parity first
cd $GRAFT_REPO_ROOT
PGPB_LIB_PATH=paper_2508_07014_b200/build/libpgpb_pf.so timeout 900 python -m pytest tests/test_ctc_fused_gpu.py tests/test_greedy_gpu.py -x -q > gpurun_out/pf_tests.log 2>&1; echo rc=$? >> gpurun_out/pf_tests.log
export PGPB_REGIMES=clean,dense,blank3 PGPB_IMPLS=fused
for rep in 1 2 3; do for lib in nopf pf; do
  echo "== $lib"; PGPB_LIB_PATH=paper_2508_07014_b200/build/libpgpb_$lib.so timeout 120 python scripts/ctc_regimes.py 2>&1 | tail -3
done; done > gpurun_out/pf_ab.log 2>&1
