"""Training step with tracking folded in (sim.py:140-155 on the GPU): one
interval of C2 (26 Criteo-Kaggle tables x d16, 500 batches x 2048 Zipf
lookups per table) applied with np.add.at semantics, with and without the
dirty-bit marking.  Prints one JSON line (device time, CUDA events)."""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2010_08679_b200 as ds  # noqa: E402
from paper_2010_08679_b200.train import apply_packed, pack_batches  # noqa: E402

dev = torch.device("cuda", 0)
cards = bench.CRITEO_KAGGLE
B, NB, D = bench.BATCH, int(os.environ.get("NB", "500")), 16
gen = torch.Generator(device=dev)
gen.manual_seed(0)
tables = {t: ds.DeviceTable(t, torch.rand((r, D), generator=gen, device=dev), None) for t, r in enumerate(cards)}
look = [bench.lookups_torch("zipf", r, NB * B, gen, dev).to(torch.int64) for r in cards]
batches = [{t: (look[t][b * B:(b + 1) * B], torch.randn((B, D), generator=gen, device=dev) * 0.01)
            for t in range(len(cards))} for b in range(NB)]
tr = ds.ModelTracker({t: r for t, r in enumerate(cards)}, device=dev)


packed = pack_batches(tables, batches)
del batches


SORTED = os.environ.get("SORTED", "1") == "1"


def run(track):
    apply_packed(tables, packed, tracker=tr if track else None, sorted_runs=SORTED)


for tr_on in (False, True):
    run(tr_on)
torch.cuda.synchronize()
res = {}
for tr_on in (False, True, False, True):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    run(tr_on)
    e1.record()
    torch.cuda.synchronize()
    res.setdefault(tr_on, []).append(e0.elapsed_time(e1))
print(json.dumps({"what": "C2 interval of training updates (np.add.at semantics), 26 tables x "
                          f"{NB} batches x {B}", "ms_untracked": min(res[False]),
                  "ms_tracked": min(res[True]),
                  "tracking_overhead_ms": min(res[True]) - min(res[False]),
                  "lookups": NB * B * len(cards), "sorted_runs": SORTED,
                  "bytes_per_interval": NB * B * len(cards) * (8 + 3 * 4 * D),
                  "GB/s": NB * B * len(cards) * (8 + 3 * 4 * D) / (min(res[True]) / 1e3) / 1e9,
                  "note": ("sorted_runs: ds_train_apply_interval (in-tree stable radix sort of "
                           "(table, row) keys, deltas gathered into sorted order, a warp per run, a "
                           "CTA per hot run); bytes = per lookup 8 (id) + 3 x 4d (delta read, row "
                           "read + write)") if SORTED else "ds_train_apply: a CTA per table, batches in order"}))
