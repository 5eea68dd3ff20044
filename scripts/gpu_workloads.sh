#!/bin/bash
# Runs on the GPU box: one bench line per BASELINE workload (device + e2e; CPU
# baseline on C2 only) into gpurun_out/w_<name>.json
mkdir -p gpurun_out
for wl in ${WORKLOADS:-C2 T T-adaptive C3 C4 C5}; do
  extra="--no-cpu"
  [ "$wl" = "C2" ] && extra=""
  timeout 900 python bench.py --workload $wl $extra --steps ${STEPS:-10} --warmup 3 > gpurun_out/w_$wl.json 2> gpurun_out/w_$wl.err
  echo "$wl rc=$?"
done
