#!/bin/bash
# ncu --set full of the T writer for each library variant given (one launch each)
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
WL=${WL:-T}
CMD="python bench.py --workload $WL --steps 2 --warmup 3 --no-e2e --no-cpu --verify-rows 0"
for v in "$@"; do
  name=$(basename ${v:-default} .so)
  DS_CUDA_LIB=$v timeout 600 $CMD > gpurun_out/plain_$name.log 2>&1; rc=$?; echo "$name plain rc=$rc"
  [ $rc -ne 0 ] && continue
  DS_CUDA_LIB=$v timeout 900 ncu --set full --clock-control none --import-source on \
      -k regex:"${NCU_K:-writer_warp}" -s ${NCU_S:-3} -c 1 -o gpurun_out/prof_${WL}_$name $CMD > gpurun_out/ncu_$name.log 2>&1
  echo "$name ncu rc=$?"
done
