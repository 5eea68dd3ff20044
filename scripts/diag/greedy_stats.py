"""Writer stats (exact decisions / exact codes / rows) and time of the
adaptive writer on random rows: python scripts/diag/greedy_stats.py [n] [d]."""
import sys
import torch
import paper_2010_08679_b200 as ds
from paper_2010_08679_b200.engine import ShardWriter, DeviceTable

n = int(sys.argv[1]) if len(sys.argv) > 1 else 200_000
d = int(sys.argv[2]) if len(sys.argv) > 2 else 128
g = torch.Generator(device="cuda").manual_seed(1)
x = torch.randn(n, d, device="cuda", generator=g)
for bw in (2, 3, 4):
    cfg = ds.quant.default_adaptive_config(bw)
    stats = torch.zeros(4, dtype=torch.int64, device="cuda")
    w = ShardWriter([DeviceTable(0, x)], bw, adaptive=cfg, stats=stats)
    pay = torch.empty(w.payload_bytes(None), dtype=torch.uint8, device="cuda")
    w.write(pay); w.finish()
    stats.zero_()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); w.write(pay); e1.record(); torch.cuda.synchronize()
    w.finish()
    print(f"bw {bw} n {n} d {d}: {e0.elapsed_time(e1):.3f} ms, {n / e0.elapsed_time(e1) / 1e3:.2f} M rows/s, "
          f"stats exact_dec {int(stats[0])} exact_codes {int(stats[1])} rows {int(stats[2])}", flush=True)
