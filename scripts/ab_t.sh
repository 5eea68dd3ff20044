#!/bin/bash
# A/B of writer variants on T and C2 (bench.py lines with parity), REPS interleaved rounds
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
REPS=${REPS:-2}
for r in $(seq $REPS); do
  for v in "$@"; do
    for wl in ${WLS:-T C2}; do
      DS_CUDA_LIB=$v timeout 600 python bench.py --workload $wl --no-cpu --no-e2e --steps ${STEPS:-10} --warmup 3 --verify-rows ${VROWS:-200000} ${BENCH_ARGS:-} > gpurun_out/ab_${wl}_$(basename ${v:-default}).json 2> gpurun_out/ab_err.txt
      python - "$v" "$wl" <<'PY'
import json,sys
v,wl=sys.argv[1],sys.argv[2]
try:
    d=json.loads(open(f"gpurun_out/ab_{wl}_{(v.split('/')[-1] if v else 'default')}.json").read().strip().splitlines()[-1])
except Exception as e:
    print(v, wl, "FAILED", e); print(open("gpurun_out/ab_err.txt").read()[-2000:]); sys.exit()
p=d['phases']; par=d.get('parity') or {}
print(f"{(v or 'default'):50s} {wl:3s} ms/step {d['ms_per_step']:.4f} " + ' '.join(f"{k} {x['ms']*1000:.1f}" for k,x in p.items()) + f" frac {d['roofline']['frac']:.3f} parity {par.get('records_checked')}/{par.get('mismatches')}")
PY
    done
  done
done
