run() { timeout 300 python scripts/bench_advance.py "$@"; }
{
PGPB_ADVANCE_VARIANT=3 run p20k_v1024 8192,65536
PGPB_ADVANCE_VARIANT=3 PGPB_V3_WARPS=4 run p20k_v1024 8192,65536
PGPB_ADVANCE_VARIANT=3 PGPB_V3_WARPS=2 run p20k_v1024 8192,65536
PGPB_ADVANCE_VARIANT=5 run p20k_v1024 1024,8192,65536
PGPB_ADVANCE_VARIANT=5 PGPB_V5_CTAS=2 run p20k_v1024 8192,65536
PGPB_ADVANCE_VARIANT=5 PGPB_V5_CTAS=1 run p20k_v1024 8192
PGPB_ADVANCE_VARIANT=5 run p20k_v4096 1024,8192
PGPB_ADVANCE_VARIANT=5 PGPB_V5_CTAS=1 run p20k_v4096 8192
} > gpurun_out/adv_sweep2.jsonl 2> gpurun_out/adv_sweep2.err
python - <<'PY'
import json
for l in open("gpurun_out/adv_sweep2.jsonl"):
    d=json.loads(l)
    print(d["variant"], d["corpus"], [(r["B"], round(r["GBps_med"]), round(r["fill_GBps"]), r["exact"]) for r in d["rows"]])
PY
tail -3 gpurun_out/adv_sweep2.err
PGPB_ADVANCE_VARIANT=5 timeout 600 python -m pytest -q -x tests/test_advance_gpu.py 2>&1 | tail -2
PGPB_ADVANCE_VARIANT=5 ncu --set full --cache-control none --clock-control none --import-source on -k regex:advance_v5 -s 6 -c 1 -o gpurun_out/prof_v5 python scripts/prof_kernels.py advance 10 > /dev/null 2>&1
PGPB_ADVANCE_VARIANT=3 ncu --set full --cache-control none --clock-control none --import-source on -k regex:advance_v3 -s 6 -c 1 -o gpurun_out/prof_v3 python scripts/prof_kernels.py advance 10 > /dev/null 2>&1
ls gpurun_out
