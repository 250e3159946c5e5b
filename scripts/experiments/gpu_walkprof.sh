cd $GRAFT_REPO_ROOT
PGPB_LIB_PATH=paper_2508_07014_b200/libpgpb_prof.so timeout 300 python scripts/ctc_fused_profile.py > gpurun_out/walkprof.log 2>&1
