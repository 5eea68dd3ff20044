"""Per-CUDA-source-line instruction and stall attribution of one kernel.

Joins ncu's SASS source page (instructions executed, stall samples per SASS
address) with `nvdisasm -g` line info of the library's cubins.

usage: python scripts/ncu_lines.py REPORT KERNEL_REGEX [TOP] [LIB]
"""
import csv, glob, io, os, re, subprocess, sys, tempfile
from collections import defaultdict

_maps = {}


def _line_maps(lib):
    """{mangled function: {offset: (file:line, sass)}} of every cubin in lib."""
    if lib in _maps:
        return _maps[lib]
    tmp = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(lib)], cwd=tmp, capture_output=True)
    fmap = {}
    for cub in glob.glob(os.path.join(tmp, "*.cubin")):
        dis = subprocess.run(["nvdisasm", "-g", "-c", cub], capture_output=True, text=True).stdout
        cur, line = None, None
        for ln in dis.splitlines():
            m = re.match(r"\s*\.text\.(\S+):", ln)
            if m:
                cur = m.group(1); fmap[cur] = {}; line = None
                continue
            m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
            if m:
                line = f"{os.path.basename(m.group(1))}:{m.group(2)}"
                continue
            m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?);", ln)
            if m and cur is not None:
                fmap[cur][int(m.group(1), 16)] = (line, m.group(2).strip())
    _maps[lib] = fmap
    return fmap


def _text(key):
    f, _, n = key.partition(":")
    path = os.path.join("paper_2010_08679_b200/csrc", f)
    if not n or not os.path.exists(path):
        return ""
    return open(path).read().splitlines()[int(n) - 1].strip()


def line_table(rep, pat, lib="paper_2010_08679_b200/libdeltasnap_cuda.so", top=25):
    """Lines of text: per-source-line share of warp instructions and stall samples."""
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{pat}"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    kname = rows[0][1]
    h = rows[1]
    ii, si = h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
    sass, seen = [], set()
    for r in rows[2:]:
        if r and r[0] in seen:
            break  # a second launch of the same kernel
        if len(r) <= si or not r[0].startswith("0x"):
            continue
        seen.add(r[0])
        sass.append((int(r[0], 16), r[1].strip(), int(r[ii] or 0), int(r[si] or 0)))
    base = sass[0][0]
    best = None
    for fn, mp in _line_maps(lib).items():
        if len(mp) < len(sass) * 0.9:
            continue
        ok = sum(1 for a, s, _, _ in sass if (a - base) in mp and
                 mp[a - base][1].split()[0] == s.split()[0]) - abs(len(mp) - len(sass))
        if best is None or ok > best[0]:
            best = (ok, fn, mp)
    ok, fn, mp = best
    agg_i, agg_s = defaultdict(int), defaultdict(int)
    for a, s, ins, st in sass:
        key = mp.get(a - base, ("?", ""))[0] or "?"
        agg_i[key] += ins
        agg_s[key] += st
    ti, ts = sum(agg_i.values()) or 1, sum(agg_s.values()) or 1
    lines = [f"{kname}", f"  matched {fn} ({ok}/{len(sass)} opcodes), {ti} warp instructions, {ts} stall samples"]
    for key in sorted(agg_i, key=lambda k: -agg_i[k])[:top]:
        lines.append(f"{agg_i[key]/ti*100:5.1f}% ins {agg_s[key]/ts*100:5.1f}% stall  {key:22s} {_text(key)[:80]}")
    return lines


if __name__ == "__main__":
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
    lib = sys.argv[4] if len(sys.argv) > 4 else "paper_2010_08679_b200/libdeltasnap_cuda.so"
    print("\n".join(line_table(sys.argv[1], sys.argv[2], lib, top)))
