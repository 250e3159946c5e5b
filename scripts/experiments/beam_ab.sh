for L in libpgpb_prev.so libpgpb.so; do
  echo "== $L"
  PGPB_LIB_PATH=$PWD/paper_2508_07014_b200/$L timeout 300 python scripts/experiments/config3_probe.py 2>&1 | tail -2
  PGPB_LIB_PATH=$PWD/paper_2508_07014_b200/$L timeout 300 python scripts/experiments/ctc_beam_probe.py 2>&1 | tail -2
done
