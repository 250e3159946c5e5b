# greedy CTC iteration: parity tests, A/B regimes vs HEAD lib
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_ctc_fused_gpu.py tests/test_greedy_gpu.py tests/test_shim_gpu.py -x -q > gpurun_out/fused_tests.log 2>&1; echo rc=$? >> gpurun_out/fused_tests.log
bash scripts/gpu_ab_ctc.sh > gpurun_out/ab.log 2>&1
