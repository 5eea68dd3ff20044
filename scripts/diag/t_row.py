"""Re-derive one T-workload row (bench.py's device draw) and compare the
writer's record for it with the oracle: python scripts/diag/t_row.py ROW"""
import sys
import numpy as np, torch
import paper_2010_08679_b200 as ds
from paper_2010_08679_b200.engine import ShardWriter, DeviceTable
sys.path.insert(0, ".")
from oracle import oracle as O

row = int(sys.argv[1])
gen = torch.Generator(device="cuda"); gen.manual_seed(0)
v = torch.rand((125_000_000, 128), generator=gen, device="cuda", dtype=torch.float32).mul_(2).sub_(1)
x = v[row:row + 1].clone(); del v
xs = x.cpu().numpy()
# 4-bit naive, full section of the one row
w = ShardWriter([DeviceTable(0, x)], 4, adaptive=None)
pay = torch.zeros(w.payload_bytes(None), dtype=torch.uint8, device="cuda")
w.write(pay); w.finish()
b = pay.cpu().numpy()[24:]
lo, hi = np.frombuffer(b[:8].tobytes(), np.float32)
codes_dev = np.unpackbits(b[8:8 + 64][None, :], axis=1, bitorder="little").reshape(-1, 4)
codes_dev = (codes_dev * (1 << np.arange(4))).sum(1)
mn, mx = O.row_minmax(xs)
codes_ref = O.quantize_rows(xs, mn, mx, 4)[0]
print("lo/hi dev", lo, hi, "ref", mn[0], mx[0])
diff = np.nonzero(codes_dev != codes_ref)[0]
print("code diffs at", diff, "dev", codes_dev[diff], "ref", codes_ref[diff], "x", xs[0, diff])
s = (np.float64(mx[0]) - np.float64(mn[0])) / 15
for i in diff:
    print(i, repr(xs[0, i]), "v_ref", (np.float64(xs[0, i]) - np.float64(mn[0])) / s)
