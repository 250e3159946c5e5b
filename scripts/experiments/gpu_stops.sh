# incremental cost of each walker stage in the real pipeline (PGPB_CTC_STOP, outputs invalid)
cd $GRAFT_REPO_ROOT
for k in 1 2 3 4 5 6 7 0; do echo "stop=$k"; PGPB_CTC_STOP=$k timeout 120 python scripts/ctc_regimes.py 2>&1 | grep clean; done
