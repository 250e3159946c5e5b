# Round profiles: bench line, bench launch list, ncu --set full of the advance kernel and both greedy-CTC kernels
cd $GRAFT_REPO_ROOT
timeout 900 python bench.py > gpurun_out/bench_full.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 600 --csv --log-file gpurun_out/r1_launches.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1
timeout 600 ncu --set full --cache-control none --clock-control none --import-source on -k regex:advance_v6 -s 6 -c 1 -o gpurun_out/r1_advance_v6 python scripts/prof_kernels.py advance 10 > gpurun_out/ncu_adv.log 2>&1
timeout 600 ncu --set full --cache-control none --clock-control none --import-source on -k regex:frame_top2 -s 2 -c 1 -o gpurun_out/r1_ctc_top2 python scripts/ctc_one.py clean > gpurun_out/ncu_ctc1.log 2>&1
timeout 600 ncu --set full --cache-control none --clock-control none --import-source on -k regex:ctc_walk -s 2 -c 1 -o gpurun_out/r1_ctc_walk python scripts/ctc_one.py clean > gpurun_out/ncu_ctc2.log 2>&1
