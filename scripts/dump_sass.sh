#!/bin/bash
# SASS listing of every kernel in the built library objects -> profiles/sass/
# (one instantiation per template: the one the benchmarks run).  Run after
# paper_2508_07014_b200/_build.py.
set -e
out=profiles/sass
mkdir -p $out
for o in paper_2508_07014_b200/build/*.o; do
  for f in $(cuobjdump -sass "$o" 2>/dev/null | grep "Function :" | awk '{print $3}'); do
    d=$(echo "$f" | c++filt | sed -e 's/(anonymous namespace):://g')
    base=$(echo "$d" | sed -e 's/<.*//' -e 's/(.*//' -e 's/^.*:://')
    targs=$(echo "$d" | sed -n 's/^[^<]*<\([^>]*\)>.*/\1/p' | sed -e 's/, /_/g' -e 's/,/_/g')
    name=$base${targs:+_$targs}
    # beams K=4 vectorised, flag pairs true/true, label loop / greedy NC=8, vectorised
    case "$targs" in ""|4_true|true_true|8|true) ;; *) continue ;; esac
    cuobjdump -sass -fun "$f" "$o" > "$out/$name.sass"
  done
done
ls $out | wc -l
