# A/B of library variants on bench workloads: LIBS="'' _x" WLS="T C1"
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
for r in $(seq ${REPS:-2}); do
for v in ${LIBS:-""}; do
  [ "$v" = "-" ] && v=""
  for wl in ${WLS:-T}; do
    DS_CUDA_LIB=$PWD/paper_2010_08679_b200/libdeltasnap_cuda$v.so timeout 600 python bench.py --workload $wl --no-cpu --no-e2e --steps ${STEPS:-10} --warmup 3 --verify-rows ${VROWS:-200000} > gpurun_out/abl.json 2> gpurun_out/abl_err.txt
    python - "lib$v" "$wl" <<'PY'
import json,sys
v,wl=sys.argv[1],sys.argv[2]
try:
    d=json.loads(open("gpurun_out/abl.json").read().strip().splitlines()[-1])
except Exception as e:
    print(v, wl, "FAILED", e); print(open("gpurun_out/abl_err.txt").read()[-3000:]); sys.exit()
p=d['phases']; par=d.get('parity') or {}
print(f"{v:18s} {wl:10s} ms/step {d['ms_per_step']:.4f} " + ' '.join(f"{k} {x['ms']*1000:.1f}" for k,x in p.items()) + f" frac {d['roofline']['frac']:.3f} parity {par.get('records_checked')}/{par.get('mismatches')}")
PY
  done
done
done
