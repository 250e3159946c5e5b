# ncu --set full of advance v6 (evict-first stores) at 8192 rows, plus the full GPU suite
cd $GRAFT_REPO_ROOT
timeout 600 ncu --set full --cache-control none --clock-control none --import-source on -k regex:advance_v6 -s 6 -c 1 -o gpurun_out/r1_advance_v6_ef python scripts/prof_kernels.py advance 10 > gpurun_out/ncu_adv.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/gpu_tests.log
