# CTC beam phase-timeline build -> paper_2508_07014_b200/libpgpb_cbprof.so
PROF_FLAG=-DPGPB_CB_PROFILE PROF_LIB=libpgpb_cbprof.so bash scripts/experiments/build_prof_lib.sh
