cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_dbeam_gpu.py tests/test_abi.py -x -q > gpurun_out/beam_tests.log 2>&1; echo rc=$? >> gpurun_out/beam_tests.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_beam.log 2>&1
