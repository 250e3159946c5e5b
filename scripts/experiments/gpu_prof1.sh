set -x
ncu --set full --clock-control none --import-source on -k regex:advance_closure -s 3 -c 1 -o gpurun_out/prof_advance python scripts/prof_kernels.py advance 6 > gpurun_out/ncu_adv.log 2>&1; tail -3 gpurun_out/ncu_adv.log
ncu --set full --clock-control none --import-source on -k regex:ctc_greedy -s 2 -c 2 -o gpurun_out/prof_greedy python scripts/prof_kernels.py greedy 4 > gpurun_out/ncu_greedy.log 2>&1; tail -3 gpurun_out/ncu_greedy.log
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,utilization.gpu,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap --format=csv,noheader,nounits 2>&1 | head -3
