# ncu --set full of the redux phase A (top-2 boosted, top-1 unboosted), clean regime; bench launch list
cd $GRAFT_REPO_ROOT
timeout 600 ncu --set full --cache-control none --clock-control none --import-source on -k regex:frame_top2 -s 2 -c 1 -o gpurun_out/r1_ctc_top2_redux python scripts/ctc_one.py clean > gpurun_out/ncu_ctc1.log 2>&1
timeout 600 ncu --set full --cache-control none --clock-control none --import-source on -k regex:frame_top2 -s 2 -c 1 -o gpurun_out/r1_ctc_top1_redux python scripts/ctc_one.py clean 0 > gpurun_out/ncu_ctc3.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 600 --csv --log-file gpurun_out/r1_launches.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1
