# advance headline: session-start configuration (cs stores, blocked rows, per-row bitmap) vs now, same box
cd $GRAFT_REPO_ROOT
for rep in 1 2 3; do for cfg in start now; do
  if [ $cfg = start ]; then E="PGPB_LIB_PATH=paper_2508_07014_b200/build/libpgpb_st0.so PGPB_V6_MAP=0 PGPB_V6_TBITS=0"; else E="X=1"; fi
  echo "== $cfg"; env $E timeout 300 python bench.py --no-decode --no-cpu-baseline 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('headline', round(d['roofline']['frac'],4), {k: round(v['frac_hbm'],4) for k,v in d.get('advance_sweep',{}).items() if isinstance(v,dict)})"
done; done > gpurun_out/adv_regress.log 2>&1
