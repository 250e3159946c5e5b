#!/bin/bash
# Round-2 measurement pass: bench (default args), the ncu launch list of a
# short bench run, and one `ncu --set full` capture of the headline kernel.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks_event_reasons.active --format=csv
timeout 600 python bench.py > gpurun_out/r2_bench.json 2> gpurun_out/r2_bench.err
tail -c 600 gpurun_out/r2_bench.err
timeout 300 python bench.py --impl reference --steps 5 --warmup 2 > gpurun_out/r2_bench_ref.json 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv \
  --log-file gpurun_out/r2_launches.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-decode \
  > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:advance_steps_compact_kernel -s 6 -c 1 \
  -o gpurun_out/r2_advance_steps python bench.py --steps 8 --warmup 3 --no-cpu-baseline --no-decode \
  > gpurun_out/r2_ncu_full.log 2>&1
tail -3 gpurun_out/r2_ncu_full.log
