# Debug build with phase-B checkpoints -> paper_2508_07014_b200/${PROF_LIB:-libpgpb_prof.so}
set -e
D=paper_2508_07014_b200
mkdir -p /tmp/pgpb_prof
for f in $D/csrc/*.cu $D/csrc/*.cpp; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo --fmad=false ${PROF_FLAG:--DPGPB_SEQ_PROFILE} \
    -Xcompiler -fPIC,-ffp-contract=off -Iinclude -I$D/csrc -c $f -o /tmp/pgpb_prof/$(basename $f).o &
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $D/${PROF_LIB:-libpgpb_prof.so} /tmp/pgpb_prof/*.o -lcudart_static -lrt -ldl -lpthread
