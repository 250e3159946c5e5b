timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
echo "B=128 ring0 $(timeout 300 python scripts/decode_sweep.py 128)"
echo "B=128 ring8 $(PGPB_CTC_RING=8 timeout 300 python scripts/decode_sweep.py 128)"
PGPB_LIB_PATH=$PWD/paper_2508_07014_b200/libpgpb_prof.so python scripts/seq_profile.py
