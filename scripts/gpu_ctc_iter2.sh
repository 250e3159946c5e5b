cd $GRAFT_REPO_ROOT
timeout 600 python scripts/ctc_sweep.py "PGPB_CTC_RING_SLOTS=0" "PGPB_CTC_RING_SLOTS=4" "PGPB_CTC_RING_SLOTS=8" "PGPB_CTC_RING_SLOTS=16" "PGPB_CTC_RING_SLOTS=16,PGPB_CTC_PRODUCERS=4" "PGPB_CTC_RING_SLOTS=16,PGPB_CTC_PRODUCERS=11" "PGPB_CTC_RING_SLOTS=0,PGPB_CTC_PRODUCERS=11" > gpurun_out/sweep.log 2>&1
PGPB_LIB_PATH=$PWD/paper_2508_07014_b200/libpgpb_prof.so timeout 300 python scripts/ctc_fused_profile.py > gpurun_out/cfprof.log 2>&1
