#!/bin/bash
# compute-sanitizer passes over scripts/sanitize_kernels.py (every libpgpb kernel once).
mkdir -p gpurun_out
export PYTORCH_NO_CUDA_MEMORY_CACHING=1
for tool in ${TOOLS:-memcheck racecheck synccheck initcheck}; do
  echo "== $tool"
  # initcheck tracks only the kernels it instruments: check every kernel so
  # torch-written inputs count as initialised; the others filter to libpgpb
  filt="--kernel-name regex=pgpb"; [ $tool = initcheck ] && filt=""
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 $filt \
    python scripts/sanitize_kernels.py > gpurun_out/r2_sanitize_$tool.log 2>&1
  echo "rc=$?"
  grep -E "ERROR SUMMARY|RACECHECK SUMMARY|sanitize workload ok|Error|error" gpurun_out/r2_sanitize_$tool.log | head -8
done
