# A/B of greedy CTC regimes: HEAD-built lib vs the working-tree lib, twice each
set -e
for i in 1 2; do
  echo "== head"; PGPB_LIB_PATH=paper_2508_07014_b200/build/libpgpb_head.so timeout 300 python scripts/ctc_regimes.py
  echo "== new"; timeout 300 python scripts/ctc_regimes.py
done
