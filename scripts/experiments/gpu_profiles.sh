ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r1_launches.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r1_launches_bench.log 2>&1; tail -1 gpurun_out/r1_launches_bench.log | head -c 200; echo
ncu --set full --cache-control none --clock-control none --import-source on -k regex:advance_v5 -s 6 -c 1 -o gpurun_out/r1_advance_v5 python scripts/prof_kernels.py advance 10 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:ctc_seq -s 1 -c 1 -o gpurun_out/r1_ctc_seq python scripts/prof_kernels.py greedy 3 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:frame_topm -s 1 -c 1 -o gpurun_out/r1_frame_topm python scripts/prof_kernels.py greedy 3 > /dev/null 2>&1
ls gpurun_out/*.ncu-rep
