#!/bin/bash
# The driver's round-end sequence on one GPU, then every workload with parity
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/f_smoke.log
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/f_gputest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/f_gputest.log
timeout 900 python bench.py > gpurun_out/f_bench.json 2> gpurun_out/f_bench.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference > gpurun_out/f_bench_ref.json 2> gpurun_out/f_bench_ref.err; echo "bench ref rc=$?"
bash scripts/gpu_workloads.sh
