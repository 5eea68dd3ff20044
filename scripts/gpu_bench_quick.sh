#!/bin/bash
# quick GPU check: gpu tests + one bench line (+ optional ncu of the named kernels)
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
timeout 300 python bench.py --no-cpu > gpurun_out/bq.json 2> gpurun_out/bq.err; echo "bench rc=$?"
python - <<'P'
import json
d=json.load(open("gpurun_out/bq.json"))
print("value", round(d["value"],1), "ms/step", round(d["ms_per_step"],4), "e2e", round(d["e2e"]["value"],1))
for k,v in d["phases"].items(): print(" ", k, {a: round(b,4) if isinstance(b,float) else b for a,b in v.items()})
print(" roofline", d["roofline"]["kernel"], round(d["roofline"]["frac"],3), "clocks", d["clocks"])
P
if [ -n "${NCU_K:-}" ]; then
  CMD="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu"
  timeout 300 $CMD > gpurun_out/plain.log 2>&1 && \
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"$NCU_K" -s ${NCU_S:-4} -c ${NCU_C:-3} \
      -o gpurun_out/prof $CMD > gpurun_out/ncu_full.log 2>&1; echo "ncu rc=$?"
fi
