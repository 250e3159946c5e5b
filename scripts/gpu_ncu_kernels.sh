#!/bin/bash
# One `ncu --set full` capture per production kernel at its bench shape
# (reports under gpurun_out/, summarised into profiles/).
mkdir -p gpurun_out
cap() {  # name workload kernel-regex skip
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$3 -s ${4:-3} -c 1 \
    -o gpurun_out/r2_$1 python scripts/ncu_workloads.py $2 > gpurun_out/r2_ncu_$1.log 2>&1
  echo "$1 rc=$? $(tail -1 gpurun_out/r2_ncu_$1.log)"
}
cap tbeam_wave config3 tbeam_wave_kernel 20
cap aed_step config4 aed_step_kernel 10
cap aed_greedy aed_greedy aed_greedy_kernel 10
cap beam_topk beam_api beam_topk_kernel 5
cap phrase_hits hits phrase_hits_kernel 0
cap label_loop label_loop label_loop_kernel 40
