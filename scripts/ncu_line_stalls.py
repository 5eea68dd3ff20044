"""Per-source-line stall reasons of one kernel (joins ncu's SASS source page
with nvdisasm line info, like ncu_lines.py).
usage: python scripts/ncu_line_stalls.py REPORT KERNEL_REGEX [TOP] [REASONS=long_sb,wait,short_sb]"""
import csv, io, subprocess, sys
from collections import defaultdict
sys.path.insert(0, "scripts")
from ncu_lines import _line_maps, _text

rep, pat = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
reasons = (sys.argv[4] if len(sys.argv) > 4 else "long_sb,wait,short_sb").split(",")
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{pat}"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
cols = {r: h.index(f"stall_{r}") for r in reasons}
sass, seen = [], set()
for r in rows[2:]:
    if r and r[0] in seen:
        break
    if len(r) < len(h) or not r[0].startswith("0x"):
        continue
    seen.add(r[0])
    sass.append((int(r[0], 16), r[1].strip(), {k: int(r[c] or 0) for k, c in cols.items()}))
base = sass[0][0]
best = None
for fn, mp in _line_maps("paper_2010_08679_b200/libdeltasnap_cuda.so").items():
    if len(mp) < len(sass) * 0.9:
        continue
    ok = sum(1 for a, s, _ in sass if (a - base) in mp and mp[a - base][1].split()[0] == s.split()[0]) - abs(len(mp) - len(sass))
    if best is None or ok > best[0]:
        best = (ok, fn, mp)
_, fn, mp = best
for reason in reasons:
    agg = defaultdict(int)
    for a, s, st in sass:
        agg[mp.get(a - base, ("?", ""))[0] or "?"] += st[reason]
    tot = sum(agg.values()) or 1
    print(f"== stall_{reason}: {tot} samples")
    for k, v in sorted(agg.items(), key=lambda t: -t[1])[:top]:
        print(f"  {100 * v / tot:5.1f}%  {k:24s} {_text(k)[:90]}")
