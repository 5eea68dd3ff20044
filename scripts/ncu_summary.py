"""Summarise an ncu report: per-kernel key metrics and top stall lines (run in the build container)."""
import csv, subprocess, sys, io
from collections import Counter

rep = sys.argv[1]
pat = sys.argv[2] if len(sys.argv) > 2 else None
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h = rows[0]
want = ['Kernel Name', 'gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed',
        'sm__throughput.avg.pct_of_peak_sustained_elapsed',
        'sm__warps_active.avg.pct_of_peak_sustained_active', 'launch__registers_per_thread',
        'launch__grid_size', 'launch__occupancy_limit_registers', 'launch__occupancy_limit_shared_mem',
        'lts__throughput.avg.pct_of_peak_sustained_elapsed',
        'l1tex__throughput.avg.pct_of_peak_sustained_active', 'smsp__inst_executed.sum',
        'sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active',
        'sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active',
        'sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active',
        'smsp__issue_active.avg.pct_of_peak_sustained_active']
idx = [h.index(w) if w in h else None for w in want]
for r in rows[2:]:
    if pat and pat not in r[h.index('Kernel Name')]:
        continue
    print('----')
    for w, i in zip(want, idx):
        if i is not None:
            print(f"  {w}: {r[i]} {rows[1][i]}")
if pat:
    src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{pat}"],
                         capture_output=True, text=True).stdout
    srows = list(csv.reader(io.StringIO(src)))
    hh = srows[1]
    si = hh.index('Warp Stall Sampling (All Samples)')
    seen, R = set(), []
    for r in srows[2:]:
        if len(r) <= si or r[0] in seen:
            continue
        seen.add(r[0]); R.append(r)
    tot = sum(int(r[si]) for r in R if r[si].isdigit()) or 1
    for r in sorted(R, key=lambda r: -int(r[si]) if r[si].isdigit() else 0)[:int(sys.argv[3]) if len(sys.argv) > 3 else 12]:
        print(f"{int(r[si])/tot*100:5.1f}%  {r[1].strip()[:90]}")
