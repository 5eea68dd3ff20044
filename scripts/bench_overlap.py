"""Checkpoints overlapped with training steps (north star item 4) on C2:
26 Criteo-Kaggle-shaped tables x d16, a training step = one batch of 2048
Zipf(1.05) lookups per table applied with np.add.at semantics and the dirty
bits marked on the fly (ds_train_apply); an interval = NB steps, then a
checkpoint through TrainingCheckpointLoop (stall: capture + dirty-row
staging; K3 from the staged copy on a side stream; pinned D2H on a copy
stream from a background thread, sim.py:329-352 / engine.py:229-233).

Prints one JSON line: the training time of an interval alone and with the
previous interval's checkpoint running beside it (slowdown), the stall, the
checkpoint's latency (stall start -> payload in pinned host memory), and a
parity check of one payload against the CPU oracle (the tables as the stall
left them).
"""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2010_08679_b200 as ds  # noqa: E402
from paper_2010_08679_b200.pipeline import TrainingCheckpointLoop  # noqa: E402
from paper_2010_08679_b200.sharded import ShardedCheckpointer  # noqa: E402
from paper_2010_08679_b200.train import apply_packed, pack_batches  # noqa: E402

NB = int(os.environ.get("NB", "100"))          # training steps per interval
POOL = int(os.environ.get("POOL", "20"))       # distinct batches cycled
INTERVALS = int(os.environ.get("INTERVALS", "6"))
B, D = bench.BATCH, 16
dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)
cards = bench.CRITEO_KAGGLE
gen = torch.Generator(device=dev)
gen.manual_seed(0)
tabs = {t: ds.DeviceTable(t, torch.rand((r, D), generator=gen, device=dev).mul_(2).sub_(1))
        for t, r in enumerate(cards)}
batches = []
for b in range(POOL):
    bt = {t: (bench.lookups_torch("zipf", r, B, gen, dev).to(torch.int64),
              torch.randn((B, D), generator=gen, device=dev) * 0.01) for t, r in enumerate(cards)}
    batches.append((bt, pack_batches(tabs, [bt])))
ck = ShardedCheckpointer([tabs[t] for t in sorted(tabs)], 8, device=dev)
dirty_cap = sum(min(r, NB * B) for r in cards)
loop = TrainingCheckpointLoop(ck, staged_rows=dirty_cap)


def train_interval(i0):
    for s in range(NB):
        apply_packed(tabs, batches[(i0 + s) % POOL][1], tracker=ck.tracker)


# warm-up (and a clean tracker)
train_interval(0)
loop.checkpoint()
loop.drain()
torch.cuda.synchronize()

# A: intervals of training alone
t_alone = []
for k in range(3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    train_interval(k * NB)
    e1.record()
    torch.cuda.synchronize()
    t_alone.append(e0.elapsed_time(e1))
ck.tracker.capture_into(ck.ids, None, fold=1)  # drop the A phase's marks
torch.cuda.synchronize()

# B: every interval ends in a checkpoint whose K3 + D2H overlap the next one
t_train, t_stall, lat = [], [], []
ends = []
done_at = {}
loop.on_payload = lambda out: done_at.setdefault(len(done_at), time.perf_counter())
parity = None
for k in range(INTERVALS):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    train_interval(k * NB)
    e1.record()
    t_host = time.perf_counter()
    stall_end = loop.checkpoint()
    if k == 1:  # parity of one payload: the tables as the stall left them
        stall_end.synchronize()
        snap = {t: (tb.values.cpu().numpy(), None) for t, tb in tabs.items()}
        sel = {}
        for t in tabs:
            ids = torch.cat([batches[(k * NB + s) % POOL][0][t][0] for s in range(NB)])
            sel[t] = np.unique(ids.cpu().numpy())
        check_k = k
    ends.append((e0, e1, stall_end, t_host))
outs = loop.drain()
torch.cuda.synchronize()
for k, (e0, e1, se, th) in enumerate(ends):
    if k:  # intervals that ran beside the previous checkpoint
        t_train.append(e0.elapsed_time(e1))
    t_stall.append(e1.elapsed_time(se))
from oracle import oracle as O  # noqa: E402
want, _, _ = O.build_shard_payload(snap, "incremental", sel, 8, sorted(tabs), nthreads=os.cpu_count())
parity = {"payloads_checked": 1, "match": outs[check_k] == want, "payload_bytes": len(want)}
loop.close()
alone = float(np.median(t_alone))
with_ck = float(np.median(t_train))
print(json.dumps({
    "what": "C2 training steps (ds_train_apply_interval per batch: in-tree stable radix sort, np.add.at "
            "semantics, dirty bits on the fly) with "
            "each interval's checkpoint (8-bit naive) running beside the next interval",
    "steps_per_interval": NB, "lookups_per_step": B * len(cards),
    "interval_train_ms_alone": alone, "interval_train_ms_with_checkpoints": with_ck,
    "training_slowdown_pct": (with_ck / alone - 1) * 100,
    "stall_ms": float(np.median(t_stall)),
    "payload_bytes_per_checkpoint": int(np.median([len(o) for o in outs])),
    "d2h_bytes_total": loop.d2h_bytes,
    "parity": parity,
}))
