cd $GRAFT_REPO_ROOT
timeout 300 python scripts/ctc_sweep.py "PGPB_CTC_TMA=1" "PGPB_CTC_TMA=0" > gpurun_out/sweep.log 2>&1
PGPB_LIB_PATH=$PWD/paper_2508_07014_b200/build/libpgpb_9d32.so timeout 300 python scripts/ctc_sweep.py "OLD=9d32" >> gpurun_out/sweep.log 2>&1
