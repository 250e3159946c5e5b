# ncu --set full of the fused label-loop step (boosted), one launch mid-decode
cd $GRAFT_REPO_ROOT
timeout 600 ncu --set full --clock-control none --import-source on -k regex:label_loop -s 40 -c 1 -o gpurun_out/r1_label_loop python scripts/rnnt_kernels.py > gpurun_out/ncu_ll.log 2>&1
