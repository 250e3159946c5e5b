#!/bin/bash
# End-of-round-2 pass after the transducer-wave changes: full GPU suite +
# smoke, the default bench line, ncu capture of the wave kernel.
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/r2g_gputest.log 2>&1
echo "pytest rc=$? $(tail -1 gpurun_out/r2g_gputest.log)"
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/r2g_bench.json 2> gpurun_out/r2g_bench.err
echo "bench rc=$?"
timeout 300 ncu --set full --clock-control none --import-source on -k regex:tbeam_wave_kernel -s 40 -c 1 \
  -o gpurun_out/r2_tbeam_wave_final python scripts/ncu_workloads.py config3 > gpurun_out/r2g_ncu_tb.log 2>&1
echo "ncu tb rc=$?"
