#!/bin/bash
# Runs on the GPU box: one bench line per BASELINE workload into
# gpurun_out/w_<name>.json (device + e2e + at-scale parity + CPU baselines).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu.csv 2>&1
lscpu > gpurun_out/lscpu.txt 2>&1
for wl in ${WORKLOADS:-C2 C1 T T-adaptive C3 C4 C5}; do
  timeout 1200 python bench.py --workload $wl --steps ${STEPS:-10} --warmup 3 ${EXTRA:-} > gpurun_out/w_$wl.json 2> gpurun_out/w_$wl.err
  echo "$wl rc=$?"
done
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/w_ref_C2.json 2> gpurun_out/w_ref_C2.err; echo "ref rc=$?"
