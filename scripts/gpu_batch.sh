#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
timeout 900 python -m pytest tests -m gpu -q -x --timeout=300 2>&1 | tail -3
SORTED=1 timeout 300 python scripts/bench_train.py
timeout 600 python scripts/bench_overlap.py
timeout 600 python bench.py --workload C5 --steps 10 --warmup 3 --verify-rows 0 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('C5', d['value'], d['ms_per_step'], d['e2e']['value'])"
