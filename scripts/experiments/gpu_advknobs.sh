# advance v6 A/B: store flavour x CTAs per SM x row map (bench sweep fractions of the HBM peak)
cd $GRAFT_REPO_ROOT
run() { echo "== $*"; env "$@" timeout 300 python bench.py --no-decode --no-cpu-baseline 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('headline', round(d['roofline']['frac'],4), {k: round(v['frac_hbm'],4) for k,v in d['advance_sweep'].items() if isinstance(v,dict)})"; }
for lib in st0 st1 st2; do run PGPB_LIB_PATH=paper_2508_07014_b200/build/libpgpb_$lib.so; done
for c in 3 5 6; do run PGPB_V6_CTAS=$c; done
run PGPB_V6_CTAS=3 PGPB_V6_MAP=1
run PGPB_V6_WARPS=8 PGPB_V6_MAP=1
for lib in st0 st1 st2; do run PGPB_LIB_PATH=paper_2508_07014_b200/build/libpgpb_$lib.so; done
