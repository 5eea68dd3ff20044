#!/bin/bash
# ncu --set full of one kernel per environment variant ("VAR=val ..." or "")
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
WL=${WL:-T}
CMD="python bench.py --workload $WL --steps 2 --warmup 3 --no-e2e --no-cpu --verify-rows 0"
i=0
for v in "$@"; do
  i=$((i+1)); name=${NAME_PREFIX:-v}$i
  env $v timeout 600 $CMD > gpurun_out/plain_$name.log 2>&1; rc=$?; echo "$name [$v] plain rc=$rc"
  [ $rc -ne 0 ] && continue
  env $v timeout 900 ncu --set full --clock-control none --import-source on \
      -k regex:"${NCU_K:-writer_}" -s ${NCU_S:-3} -c 1 -o gpurun_out/prof_${WL}_$name $CMD > gpurun_out/ncu_$name.log 2>&1
  echo "$name ncu rc=$?"
done
