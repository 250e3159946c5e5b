# fused RNN-T iteration: parity (replay) tests, then the config-2 bench line
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_rnnt_gpu.py tests/test_greedy_gpu.py tests/test_abi.py tests/test_ctc_fused_gpu.py tests/test_shim_gpu.py -x -q > gpurun_out/rnnt_tests.log 2>&1; echo rc=$? >> gpurun_out/rnnt_tests.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_rnnt.log 2>&1
