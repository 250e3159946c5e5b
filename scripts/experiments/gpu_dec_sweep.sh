timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
for r in 8 2 0; do echo "ring=$r $(PGPB_CTC_RING=$r timeout 300 python scripts/decode_sweep.py 128)"; done
echo "B=1024 $(timeout 300 python scripts/decode_sweep.py 1024)"
