cd $GRAFT_REPO_ROOT
for lib in head rx; do echo "== $lib"; PGPB_LIB_PATH=paper_2508_07014_b200/build/libpgpb_$lib.so timeout 600 python -m pytest tests/test_ctc_fused_gpu.py -q -k ties 2>&1 | grep -E "^E   .*Assert|passed|failed"; done > gpurun_out/ties.log 2>&1
