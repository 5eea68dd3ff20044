"""Rank program of tests/test_multi_gpu.py (torchrun, NCCL, one GPU per rank).

Each rank holds contiguous row shards of every table, marks its share of a
global Zipf-like lookup stream, runs K2 + the count exchange (NVLink peer
stores, or the NCCL all_gather with DS_COUNTS_EXCHANGE=nccl) + K3
(ShardedCheckpointer.step; the second of three intervals staged), and rank 0
assembles the shard payload from every rank's D2H'd runs.  It must equal the oracle's single-process payload of the
whole tables (engine.py:118-189) byte for byte.
"""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402  (test infrastructure: the checker)
from paper_2010_08679_b200.sharded import ShardedCheckpointer, make_local_tables, shard_rows  # noqa: E402

ROWS = {0: 200_003, 1: 5_000, 2: 1_000_000, 3: 17}


def main():
    bitwidth = int(sys.argv[1]) if len(sys.argv) > 1 and sys.argv[1] != "fp32" else None
    dim = int(sys.argv[2]) if len(sys.argv) > 2 else 16
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    rng = np.random.default_rng(42)
    full = {t: rng.standard_normal((r, dim)).astype(np.float32) for t, r in ROWS.items()}
    shapes = {t: (r, dim) for t, r in ROWS.items()}

    def init(tid, lo, v):
        v.copy_(torch.from_numpy(full[tid][lo:lo + v.shape[0]]))

    tables = make_local_tables(shapes, world, rank, dev, init)
    ck = ShardedCheckpointer(tables, bitwidth, rank=rank, world_size=world, device=dev)
    want_peer = os.environ.get("DS_COUNTS_EXCHANGE", "peer") != "nccl"
    assert (ck._peer is not None) == want_peer, "count exchange transport"
    # three intervals (exchange epochs 1..3, both slot parities); the second
    # one through stall-window staging
    ok = True
    for interval in range(3):
        look = {t: np.minimum(rng.zipf(1.2, 50_000) - 1, r - 1).astype(np.int64) for t, r in ROWS.items()}
        idx, seg = [], [0]
        for t in sorted(ROWS):
            lo, hi = shard_rows(ROWS[t], world, rank)
            mine = look[t][(look[t] >= lo) & (look[t] < hi)] - lo
            idx.append(mine)
            seg.append(seg[-1] + mine.size)
        sel = {}  # this rank's dirty rows, global ids
        for k, t in enumerate(sorted(ROWS)):
            lo, hi = shard_rows(ROWS[t], world, rank)
            sel[t] = np.unique(idx[k]) + lo
        ids = torch.from_numpy(np.concatenate(idx)).to(torch.int32).to(dev)
        if interval == 1:
            ck.mark(ids, np.array(seg), np.arange(len(ROWS)))
            ck.checkpoint(staged_rows=sum(ROWS.values()))
        else:
            ck.step(ids, np.array(seg), np.arange(len(ROWS)))
        torch.cuda.synchronize()
        buf, n = ck.fetch()
        torch.cuda.synchronize()
        _, local_counts, per_table, _, _ = ck.layout()
        mine = (bytes(buf[:n].numpy()), np.asarray(local_counts).copy())
        got = [None] * world
        dist.all_gather_object(got, mine)
        sels = [None] * world
        dist.all_gather_object(sels, sel)
        if rank == 0:
            blob = ck.assemble(got, per_table)
            gsel = {t: np.sort(np.concatenate([s[t] for s in sels])) for t in ROWS}
            ref, _, _ = O.build_shard_payload({t: (full[t], None) for t in ROWS}, "incremental", gsel,
                                              bitwidth, sorted(ROWS))
            if blob != ref:
                ok = False
                print(f"MISMATCH interval {interval}: {len(blob)} {len(ref)}", flush=True)
    if rank == 0 and ok:
        print("OK", flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
