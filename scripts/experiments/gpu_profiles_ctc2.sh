cd $GRAFT_REPO_ROOT
timeout 600 ncu --set full --clock-control none --import-source on -k regex:frame_top2 -s 2 -c 1 -o gpurun_out/r1_ctc_top2 python scripts/ctc_one.py clean > gpurun_out/ncu_ctc1.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:frame_top2 -s 2 -c 1 -o gpurun_out/r1_ctc_top1 python scripts/ctc_one.py clean 0 > gpurun_out/ncu_ctc3.log 2>&1
