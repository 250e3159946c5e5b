#!/bin/bash
# ncu captures of the kernels not covered by gpu_ncu_kernels.sh / the headline capture.
mkdir -p gpurun_out
cap() {  # name workload kernel-regex skip
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$3 -s ${4:-0} -c 1 \
    -o gpurun_out/r2_$1 python scripts/ncu_workloads.py $2 > gpurun_out/r2_ncu_$1.log 2>&1
  echo "$1 rc=$? $(tail -1 gpurun_out/r2_ncu_$1.log)"
}
cap frame_top2 ctc_clean_boosted frame_top2_kernel 2
cap ctc_walk ctc_clean_boosted ctc_walk_kernel 2
cap advance_v6 advance_single advance_v6_kernel 2
cap joint_hidden label_loop joint_hidden_kernel 20
cap lstm_update label_loop lstm_update_kernel 20
cap greedy_step greedy_host greedy_step_kernel 5
cap beam_hidden config3 beam_hidden_kernel 0
cap row_max table_helpers row_max_kernel 0
cap backoff_total table_helpers backoff_total_kernel 0
