cd $GRAFT_REPO_ROOT
for v in 6 8; do
PGPB_ADVANCE_VARIANT=$v timeout 600 ncu --set full --clock-control none --import-source on -k regex:advance_v -s 5 -c 1 -o gpurun_out/adv_v$v python bench.py --no-decode --no-cpu-baseline --steps 3 --warmup 3 > gpurun_out/ncu_adv$v.log 2>&1
done
