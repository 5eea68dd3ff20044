#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
rm -rf gpurun_out/*.ncu-rep
bash scripts/gpu_profile_r02.sh
du -sh gpurun_out
