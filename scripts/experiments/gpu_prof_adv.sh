# ncu capture of the production advance kernel (v6), same protocol as round-1 v5
cd $GRAFT_REPO_ROOT
timeout 600 ncu --set full --cache-control none --clock-control none --import-source on -k regex:advance_v6 -s 6 -c 1 -o gpurun_out/r1_advance_v6 python scripts/prof_kernels.py advance 10 > gpurun_out/ncu_adv.log 2>&1
