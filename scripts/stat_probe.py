import torch, numpy as np, sys
sys.path.insert(0, '.')
import paper_2010_08679_b200 as ds
dev = torch.device('cuda', 0)
g = torch.Generator(device=dev); g.manual_seed(0)
for kind in ("rand", "normal"):
    v = torch.rand((1_000_000, 16), generator=g, device=dev).mul_(2).sub_(1) if kind == "rand" else torch.randn((1_000_000, 16), generator=g, device=dev)
    t = ds.DeviceTable(0, v)
    stats = torch.zeros(4, dtype=torch.int64, device=dev)
    w = ds.ShardWriter([t], 8, device=dev, stats=stats)
    out = torch.empty(w.payload_bytes(None) + 16, dtype=torch.uint8, device=dev)
    w.write(out)
    w.finish()
    s = stats.cpu().numpy()
    print(kind, "exact codes", s[1], "rows", s[2], "frac elems", s[1] / (s[2] * 16))
