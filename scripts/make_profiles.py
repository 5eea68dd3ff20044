"""Write profiles/<tag>_summary.md (+ traffic.json) from a gpu_profile.sh run in gpurun_out/.

usage: python scripts/make_profiles.py r01
"""
import csv, io, json, os, subprocess, sys
from collections import OrderedDict

sys.path.insert(0, os.path.dirname(__file__))
import ncu_lines  # noqa: E402

tag = sys.argv[1]
workload = sys.argv[2] if len(sys.argv) > 2 else "C2"
G = "gpurun_out"
out = []
b = json.load(open(f"{G}/bench.json"))
out.append(f"# {tag}: profile summary\n")
out.append("## bench.py (default run, N=1)\n")
out.append("```json\n" + json.dumps(b, indent=1) + "\n```\n")
if os.path.exists(f"{G}/bench_ref.json"):
    out.append("## bench.py --impl reference\n")
    out.append("```json\n" + open(f"{G}/bench_ref.json").read().strip() + "\n```\n")
if os.path.exists(f"{G}/lscpu.txt"):
    cpu = [l for l in open(f"{G}/lscpu.txt") if l.startswith(("Model name", "CPU(s)"))]
    out.append("Host: " + "; ".join(l.split(":", 1)[0] + ": " + l.split(":", 1)[1].strip() for l in cpu) + "\n")

# launch list (ncu --metrics gpu__time_duration.sum, cold-cache, serialised)
if os.path.exists(f"{G}/launches.csv"):
    rows = [r for r in csv.reader(open(f"{G}/launches.csv")) if len(r) > 10]
    h = rows[0]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    agg = OrderedDict()
    for r in rows[1:]:
        agg.setdefault(r[ki].split("(")[0].replace("void ", ""), []).append(float(r[vi].replace(",", "")))
    tot = sum(sum(v) for v in agg.values())
    out.append("## ncu launch list (our kernels, gpu__time_duration.sum, --clock-control none)\n")
    out.append("| kernel | launches | mean µs | share |\n|---|---|---|---|")
    for k, v in agg.items():
        out.append(f"| `{k}` | {len(v)} | {sum(v)/len(v)/1e3:.1f} | {sum(v)/tot*100:.1f}% |")
    out.append("")

# full capture: key counters per kernel + per-line attribution
raw = subprocess.run(["ncu", "-i", f"{G}/prof.ncu-rep", "--page", "raw", "--csv"],
                     capture_output=True, text=True).stdout
R = list(csv.reader(io.StringIO(raw)))
h, units = R[0], R[1]
keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "smsp__inst_executed.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "sm__cycles_active.avg", "sm__cycles_active.max",
        "lts__t_sectors_srcunit_tex_op_red.sum"]
traffic = {}
seen = set()
out.append("## ncu --set full (one launch per kernel)\n")
for r in R[2:]:
    name = r[h.index("Kernel Name")]
    short = name.split("(")[0].replace("void ", "")
    if short in seen:
        continue
    seen.add(short)
    out.append(f"### `{short}`\n")
    out.append("| metric | value |\n|---|---|")
    for k in keys:
        if k in h:
            out.append(f"| {k} | {r[h.index(k)]} {units[h.index(k)]} |")
    rd = float(r[h.index("dram__bytes_read.sum")]) * (1e6 if "Mbyte" in units[h.index("dram__bytes_read.sum")] else 1)
    wr = float(r[h.index("dram__bytes_write.sum")]) * (1e6 if "Mbyte" in units[h.index("dram__bytes_write.sum")] else 1)
    if "mark_tma" in short:
        traffic["mark"] = rd + wr
    if "writer" in short:
        traffic["write"] = rd + wr
    out.append("")
    pat = short.split("<")[0].split("::")[-1]
    try:
        lines = ncu_lines.line_table(f"{G}/prof.ncu-rep", pat, top=15)
        out.append("Top source lines (share of warp instructions / stall samples):\n```\n" +
                   "\n".join(lines) + "\n```\n")
    except Exception as e:  # noqa: BLE001
        out.append(f"(line attribution failed: {e})\n")
os.makedirs("profiles", exist_ok=True)
open(f"profiles/{tag}_summary.md", "w").write("\n".join(out) + "\n")
tp = "profiles/traffic.json"
allt = json.load(open(tp)) if os.path.exists(tp) else {}
allt = {k: v for k, v in allt.items() if isinstance(v, dict)}  # per-workload entries
allt[workload] = traffic
json.dump(allt, open(tp, "w"), indent=1)
print(f"wrote profiles/{tag}_summary.md", traffic)
