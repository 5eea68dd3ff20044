"""profiles/<tag>_workloads.md from gpu_workloads.sh output (gpurun_out/w_*.json)."""
import json, os, sys

tag = sys.argv[1]
rows, raw = [], []
for wl in ["C2", "T", "T-adaptive", "C3", "C4", "C5"]:
    p = f"gpurun_out/w_{wl}.json"
    if not os.path.exists(p):
        continue
    try:
        d = json.load(open(p))
    except Exception:
        continue
    raw.append((wl, d))
    ph = d.get("phases", {})
    fmt = lambda k: (f"{ph[k]['ms']*1e3:.1f} µs" if ph[k]['ms'] < 1 else f"{ph[k]['ms']:.2f} ms") if k in ph else "–"
    rows.append(f"| {wl} | {d['value']:.1f} | {d['ms_per_step']:.3f} | {fmt('mark')} | {fmt('capture')} | "
                f"{fmt('write')} | {d['roofline']['achieved']:.0f} ({100*d['roofline']['frac']:.1f}%) | "
                f"{d['e2e']['value']:.1f} | "
                f"{(str(round(d['cpu_baseline']['value'], 3)) + ' (' + str(d['cpu_baseline']['cores']) + ' cores)') if d.get('cpu_baseline') else '–'} |")
out = [f"# {tag}: every BASELINE workload on one B200", "",
       "`bash scripts/gpu_workloads.sh` (bench.py --workload W). value = checkpointed (C5: restored) "
       "fp32 row GB/s, device-timed with L2 flushed between steps; roofline = algorithmic bytes of the "
       "dominant phase / its time vs the measured 6445 GB/s; e2e = the same through the public API "
       "with host buffers (lookups H2D, payload D2H).", "",
       "| workload | value GB/s | ms/step | mark | capture | write / restore | roofline GB/s (frac) | e2e GB/s | CPU oracle GB/s |",
       "|---|---|---|---|---|---|---|---|---|"] + rows + ["", "## raw lines", ""]
for wl, d in raw:
    out.append(f"### {wl}\n```json\n{json.dumps(d)}\n```\n")
open(f"profiles/{tag}_workloads.md", "w").write("\n".join(out) + "\n")
print("\n".join(out[:12 + len(rows)]))
