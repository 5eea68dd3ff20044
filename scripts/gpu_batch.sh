#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_scale_parity.py -m gpu -q -x --timeout=300 2>&1 | tail -2
REPS=2 WLS="C2 C1 T" STEPS=20 VROWS=100000 BENCH_ARGS="--no-shipped" bash scripts/ab_env.sh "" "DS_CUDA_LIB=paper_2010_08679_b200/libdeltasnap_cuda_me0.so"
