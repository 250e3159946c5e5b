# build_var.sh OUT.so EXTRA_FLAGS
set -e
OUT=$1; shift
D=$(mktemp -d)
for f in paper_2508_07014_b200/csrc/*.cu paper_2508_07014_b200/csrc/*.cpp; do
  b=$(basename $f)
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo --fmad=false "$@" \
    -Xcompiler -fPIC,-ffp-contract=off -Iinclude -Ipaper_2508_07014_b200/csrc -c "$f" -o "$D/$b.o" &
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o "$OUT" "$D"/*.o -lcudart_static -lrt -ldl -lpthread
rm -rf "$D"
