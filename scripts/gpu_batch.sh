#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x --timeout=300 -k "apply_batches or interval_training or sort_pairs or overlapped" 2>&1 | tail -4
SORTED=1 timeout 300 python scripts/bench_train.py
timeout 600 python scripts/bench_overlap.py
NB=500 SORTED=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"sort_|train_" --csv python scripts/bench_train.py 2>&1 | grep -E "sort_|train_" | awk -F'","' '{print $5, $(NF)}' | sort | uniq -c | sort -rn | head -12
