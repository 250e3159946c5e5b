# round-0 cost under table-load experiments (PGPB_CTC_EXP)
cd $GRAFT_REPO_ROOT
for e in 0 4 3; do for k in 4 5; do echo "exp=$e stop=$k"; PGPB_CTC_EXP=$e PGPB_CTC_STOP=$k timeout 120 python scripts/ctc_regimes.py 2>&1 | grep clean; done; done
