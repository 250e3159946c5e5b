# Build libpgpb.so from the csrc/ of a git revision (A/B timing): build_rev_lib.sh REV OUT.so
set -e
REV=$1; OUT=$2
D=$(mktemp -d)
git archive "$REV" paper_2508_07014_b200/csrc include | tar -x -C "$D"
for f in "$D"/paper_2508_07014_b200/csrc/*.cu "$D"/paper_2508_07014_b200/csrc/*.cpp; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo --fmad=false \
    -Xcompiler -fPIC,-ffp-contract=off -I"$D"/include -I"$D"/paper_2508_07014_b200/csrc -c "$f" -o "$f.o" &
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o "$OUT" "$D"/paper_2508_07014_b200/csrc/*.o -lcudart_static -lrt -ldl -lpthread
rm -rf "$D"
