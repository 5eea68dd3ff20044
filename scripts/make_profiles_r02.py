"""profiles/<tag>_ncu.md + profiles/traffic.json from scripts/gpu_profile_r02.sh
output in gpurun_out/ (p_<name>_launches.csv, p_<name>.ncu-rep).

usage: python scripts/make_profiles_r02.py r02
"""
import csv, io, json, os, subprocess, sys
from collections import OrderedDict

sys.path.insert(0, os.path.dirname(__file__))
import ncu_lines  # noqa: E402

tag = sys.argv[1]
G = "gpurun_out"
PO = os.environ.get("PROFILE_OUT", "profiles")  # gpurun_out on the box (only it travels back)
TP = os.environ.get("TRAFFIC_IN", "profiles/traffic.json")
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "smsp__inst_executed.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"]
WHAT = {"C2": "bench.py (C2, default): K1 mark, K2 capture, K3 writer",
        "T": "bench.py --workload T: the north-star shard's writer (125M x 128, 4-bit naive)",
        "C4": "bench.py --workload C4: adaptive greedy writer (2-bit, 25 evaluations per row)",
        "C5": "bench.py --workload C5: restore of a 1 full + 5 incremental chain",
        "train": "scripts/bench_train.py: one C2 interval of training updates (in-tree sort path)"}
out = [f"# {tag}: ncu (B200, --clock-control none)", "",
       "Launch lists: `ncu --metrics gpu__time_duration.sum` of the plain command (cold-cache, "
       "serialised: the kernels' SHARES are what compare with the bench's phases). Full captures: "
       "`ncu --set full --import-source on`, one launch per kernel; per-line attribution by "
       "`scripts/ncu_lines.py`.", ""]
traffic = json.load(open(TP)) if os.path.exists(TP) else {}
for name in ["C2", "T", "C4", "C5", "train"]:
    lp = f"{G}/p_{name}_launches.csv"
    rp = f"{G}/p_{name}.ncu-rep"
    if not os.path.exists(lp) and not os.path.exists(rp):
        continue
    out.append(f"## {name}: {WHAT[name]}\n")
    if os.path.exists(lp):
        rows = [r for r in csv.reader(open(lp)) if len(r) > 10]
        if rows:
            h = rows[0]
            ki, vi = h.index("Kernel Name"), h.index("Metric Value")
            agg = OrderedDict()
            for r in rows[1:]:
                agg.setdefault(r[ki].split("(")[0].replace("void ", ""), []).append(
                    float(r[vi].replace(",", "")))
            tot = sum(sum(v) for v in agg.values())
            out.append("| kernel | launches | mean µs | share |\n|---|---|---|---|")
            for k, v in agg.items():
                out.append(f"| `{k}` | {len(v)} | {sum(v)/len(v)/1e3:.1f} | {sum(v)/tot*100:.1f}% |")
            out.append("")
    if not os.path.exists(rp):
        continue
    raw = subprocess.run(["ncu", "-i", rp, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    R = list(csv.reader(io.StringIO(raw)))
    if len(R) < 3:
        continue
    h, units = R[0], R[1]
    seen = {}
    dram_sum = 0.0
    for r in R[2:]:
        short = r[h.index("Kernel Name")].split("(")[0].replace("void ", "")
        b = sum(float(r[h.index(k)]) * UNIT.get(units[h.index(k)], 1)
                for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
        dram_sum += b
        if short in seen:
            continue
        seen[short] = b
        out.append(f"### `{short}`\n")
        out.append("| metric | value |\n|---|---|")
        for k in KEYS:
            if k in h:
                out.append(f"| {k} | {r[h.index(k)]} {units[h.index(k)]} |")
        out.append("")
        pat = short.split("<")[0].split("::")[-1]
        try:
            lines = ncu_lines.line_table(rp, pat, top=18)
            out.append("Top source lines (share of warp instructions / stall samples):\n```\n" +
                       "\n".join(lines) + "\n```\n")
        except Exception as e:  # noqa: BLE001
            out.append(f"(line attribution failed: {e})\n")
    t = traffic.setdefault(name, {}) if name != "train" else {}
    for short, b in seen.items():
        if "mark_tma" in short:
            t["mark"] = b
        if "writer" in short:
            t["write"] = b
    if name == "C5":
        t["restore_chain"] = dram_sum  # the 6 captured launches = one chain
    if name != "train":
        traffic[name] = t
open(f"{PO}/{tag}_ncu.md", "w").write("\n".join(out) + "\n")
json.dump(traffic, open(f"{PO}/traffic.json", "w"), indent=1)
print(json.dumps(traffic, indent=1))
