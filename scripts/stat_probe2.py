"""Exact-fallback rates of the certified greedy search (ShardWriter stats)."""
import sys, os, json
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2010_08679_b200 as ds
from paper_2010_08679_b200.engine import ShardWriter
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev); g.manual_seed(0)
rows = 1_000_000
vals = torch.rand((rows, 128), generator=g, device=dev).mul_(2).sub_(1)
t = ds.DeviceTable(0, vals)
for bw, cfg in ((2, (25, 0.5)), (3, (25, 0.2)), (4, (45, 0.2))):
    stats = torch.zeros(4, dtype=torch.int64, device=dev)
    acfg = ds.AdaptiveConfig(*cfg)
    w = ShardWriter([t], bw, adaptive=acfg, stats=stats)
    buf = torch.empty(w.payload_bytes(None) + 16, dtype=torch.uint8, device=dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    w.write(buf); torch.cuda.synchronize()
    stats.zero_()
    e0.record(); w.write(buf); e1.record(); w.finish()
    s = stats.cpu().numpy()
    steps = acfg.steps
    print(json.dumps({"bits": bw, "ms": e0.elapsed_time(e1), "rows": int(s[2]),
                      "exact_decisions": int(s[0]), "decisions": rows * steps * 2,
                      "frac_exact": float(s[0]) / (rows * steps * 2), "exact_codes": int(s[1])}))
