cd "${GRAFT_REPO_ROOT:-/root/repo}"
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -4
REPS=1 WLS="C2 T C4" bash scripts/ab_env.sh "" "DS_ROW_G=0" "DS_CUDA_LIB=paper_2010_08679_b200/libdeltasnap_cuda_nofuse.so DS_ROW_G=0"
for s in 0 1; do SORTED=$s timeout 300 python scripts/bench_train.py; done
timeout 600 python scripts/bench_overlap.py
