cd $GRAFT_REPO_ROOT
for e in 0 7; do echo "exp=$e stop=1"; PGPB_CTC_EXP=$e PGPB_CTC_STOP=1 timeout 120 python scripts/ctc_regimes.py 2>&1 | grep clean; done
echo "pdl0 stop=1"; PGPB_CTC_PDL=0 PGPB_CTC_STOP=1 timeout 120 python scripts/ctc_regimes.py 2>&1 | grep clean
echo "pdl0 stop=0"; PGPB_CTC_PDL=0 timeout 120 python scripts/ctc_regimes.py 2>&1 | grep clean
