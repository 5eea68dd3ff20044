#!/bin/bash
# one GPU round trip: smoke, the -m gpu suite (no -x: every failure), the default bench line
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
nvidia-smi -L > gpurun_out/gpus.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout ${TEST_TIMEOUT:-1800} python -m pytest tests -m gpu -q ${PYTEST_ARGS:-} > gpurun_out/gputest.log 2>&1; echo "pytest rc=$?"
tail -30 gpurun_out/gputest.log
if [ -z "$NO_BENCH" ]; then
  timeout 900 python bench.py ${BENCH_ARGS:---steps 20 --warmup 5} > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
  tail -c 3000 gpurun_out/bench.json; tail -5 gpurun_out/bench.err
fi
