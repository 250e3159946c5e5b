cd $GRAFT_REPO_ROOT
timeout 600 python scripts/ctc_sweep.py "PGPB_CTC_PDL=1" "PGPB_CTC_PDL=0" > gpurun_out/sweep.log 2>&1
