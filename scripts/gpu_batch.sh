#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
REPS=1 WLS="C4 C3" VROWS=300000 BENCH_ARGS="--no-shipped" bash scripts/ab_env.sh "" "DS_CUDA_LIB=paper_2010_08679_b200/libdeltasnap_cuda_noties.so"
