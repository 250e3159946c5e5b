cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_rnnt_gpu.py tests/test_greedy_gpu.py tests/test_ctc_fused_gpu.py tests/test_shim_gpu.py tests/test_beam_gpu.py -x -q > gpurun_out/rnnt_tests.log 2>&1; echo rc=$? >> gpurun_out/rnnt_tests.log
for i in 1 2; do timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_rnnt$i.log 2>&1; done
