cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_ctc_fused_gpu.py tests/test_greedy_gpu.py -x -q > gpurun_out/fused_tests.log 2>&1; echo rc=$? >> gpurun_out/fused_tests.log
for i in 1 2; do for w in 4 7; do echo "W=$w"; PGPB_CTC_CONSUMERS=$w timeout 120 python scripts/ctc_regimes.py 2>&1 | grep -v Warn; done; done > gpurun_out/abw.log 2>&1
