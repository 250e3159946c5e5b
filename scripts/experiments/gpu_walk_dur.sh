# serialized kernel durations of one boosted greedy-CTC call per regime (ncu, warm L2): HEAD lib vs working tree
cd $GRAFT_REPO_ROOT
for lib in build/libpgpb_head.so libpgpb.so; do
  for r in clean blank3; do
    PGPB_LIB_PATH=paper_2508_07014_b200/$lib timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none \
      -k regex:"ctc_walk|frame_top2" --csv python scripts/ctc_one.py $r 2>/dev/null | grep -E "ctc_walk|frame_top2" | \
      awk -F'","' -v L=$lib -v R=$r '{print L, R, $5, $NF}'
  done
done
