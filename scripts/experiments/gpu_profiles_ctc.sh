# ncu captures for the greedy CTC kernels (clean regime, B=128 x 200, 20K tree)
cd $GRAFT_REPO_ROOT
timeout 600 ncu --set full --clock-control none --import-source on -k regex:frame_top2 -s 4 -c 1 -o gpurun_out/r1_ctc_top2 python scripts/ctc_one.py clean > gpurun_out/ncu_ctc1.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:ctc_walk -s 2 -c 1 -o gpurun_out/r1_ctc_walk python scripts/ctc_one.py clean > gpurun_out/ncu_ctc2.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:frame_top2 -s 4 -c 1 -o gpurun_out/r1_ctc_top1 python scripts/ctc_one.py clean 0 > gpurun_out/ncu_ctc3.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 600 --csv --log-file gpurun_out/r1_launches.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1
cuobjdump -sass -fun frame_top2_kernel paper_2508_07014_b200/libpgpb.so > gpurun_out/sass_top2.txt 2>&1 || true
