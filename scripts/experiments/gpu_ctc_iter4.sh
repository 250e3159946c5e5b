# greedy CTC iteration: parity tests (CTC, greedy, shim, hits, GPB1), A/B regimes vs HEAD lib, per-stage costs
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_ctc_fused_gpu.py tests/test_greedy_gpu.py tests/test_shim_gpu.py tests/test_hits.py tests/test_gpb1_device.py -x -q > gpurun_out/fused_tests.log 2>&1; echo rc=$? >> gpurun_out/fused_tests.log
bash scripts/gpu_ab_ctc.sh > gpurun_out/ab.log 2>&1
bash scripts/gpu_stops.sh > gpurun_out/stops.log 2>&1
