# greedy CTC iteration: parity tests, A/B regimes vs HEAD lib, CTA-0 timeline
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_ctc_fused_gpu.py tests/test_greedy_gpu.py tests/test_shim_gpu.py -x -q > gpurun_out/fused_tests.log 2>&1; echo rc=$? >> gpurun_out/fused_tests.log
bash scripts/gpu_ab_ctc.sh > gpurun_out/ab.log 2>&1
PGPB_LIB_PATH=$PWD/paper_2508_07014_b200/libpgpb_prof.so timeout 300 python scripts/ctc_fused_profile.py > gpurun_out/cfprof.log 2>&1
