"""profiles/<tag>_workloads.md from gpu_workloads.sh output (gpurun_out/w_*.json)."""
import json, os, sys

tag = sys.argv[1]
rows, raw = [], []


def last_json(p):
    return json.loads(open(p).read().strip().splitlines()[-1])


for wl in ["C2", "C1", "T", "T-adaptive", "C3", "C4", "C5"]:
    p = f"gpurun_out/w_{wl}.json"
    if not os.path.exists(p):
        continue
    try:
        d = last_json(p)
    except Exception:
        continue
    raw.append((wl, d))
    ph = d.get("phases", {})
    fmt = lambda k: (f"{ph[k]['ms']*1e3:.1f} µs" if ph[k]['ms'] < 1 else f"{ph[k]['ms']:.2f} ms") if k in ph else "–"
    cpu = d.get("cpu_baseline") or {}
    sh = cpu.get("reference_as_shipped") or {}
    par = d.get("parity") or {}
    e2e = d.get("e2e") or {}
    pk = (e2e.get("packed_stream") or {}).get("value")
    rows.append(
        f"| {wl} | {d['value']:.1f} | {d['ms_per_step']:.3f} | {fmt('mark')} | {fmt('capture')} | "
        f"{fmt('write')} | {d['roofline']['achieved']:.0f} ({100*d['roofline']['frac']:.1f}%) | "
        f"{e2e.get('value', 0):.1f}{' / ' + format(pk, '.1f') if pk else ''} | "
        f"{(format(cpu['value'], '.3f') + ' (' + str(cpu['cores']) + ' thr)') if cpu else '–'} | "
        f"{(format(sh['value'], '.4f') + ' (1 thr)') if sh else '–'} | "
        f"{(par.get('records_checked') or par.get('rows_checked') or 0):,} / {par.get('mismatches', '–')} |")
out = [f"# {tag}: every BASELINE workload on one B200", "",
       "`bash scripts/gpu_workloads.sh` (bench.py --workload W). value = checkpointed (C5: restored) "
       "fp32 row GB/s, device-timed with L2 flushed between steps; roofline = algorithmic bytes of the "
       "dominant phase / its time vs the measured HBM copy bandwidth (MEASURED_PEAKS.json); e2e = the "
       "same through the public API with host buffers (int32 lookups H2D / bit-packed LookupStream "
       "H2D, payload D2H); CPU = the oracle port on all host threads (kind port) and the reference "
       "package as shipped (baseline/_ref, one writer thread); parity = records re-derived by the "
       "CPU oracle at full scale (plus every header and the whole dirty-id column) / mismatches.", "",
       "| workload | value GB/s | ms/step | mark | capture | write / restore | roofline GB/s (frac) | "
       "e2e GB/s (int32 / packed) | CPU port GB/s | reference as shipped GB/s | parity records / mismatches |",
       "|---|---|---|---|---|---|---|---|---|---|---|"] + rows + ["", "## raw lines", ""]
for wl, d in raw:
    out.append(f"### {wl}\n```json\n{json.dumps(d)}\n```\n")
if os.path.exists("gpurun_out/w_ref_C2.json"):
    out.append(f"### --impl reference (C2)\n```json\n{json.dumps(last_json('gpurun_out/w_ref_C2.json'))}\n```\n")
open(f"profiles/{tag}_workloads.md", "w").write("\n".join(out) + "\n")
print("\n".join(out[:12 + len(rows)]))
