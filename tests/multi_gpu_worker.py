"""Rank program of tests/test_multi_gpu.py (torchrun, NCCL, one GPU per rank).

Each rank holds contiguous row shards of every table, marks its share of a
global Zipf-like lookup stream, runs K2 + the count exchange (NVLink peer
stores, or the NCCL all_gather with DS_COUNTS_EXCHANGE=nccl) + K3
(ShardedCheckpointer.step; the second of three intervals staged), and rank 0
assembles the shard payload from every rank's D2H'd runs.  It must equal the oracle's single-process payload of the
whole tables (engine.py:118-189) byte for byte.  Then every rank restores
its rows of a full + 2 incremental chain from rank-local uploads
(engine.rank_slices) and checks them against the oracle's restore.
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
    # rank-local restore of a full + 2 incremental chain (SURVEY 8(e) "Restore"):
    # every rank restores its rows, uploading only its records; its rows and
    # since-baseline bits equal the oracle's restore of the whole chain
    if bitwidth is not None:
        import paper_2010_08679_b200 as ds
        from paper_2010_08679_b200.engine import apply_payload
        vals = {t: v.copy() for t, v in full.items()}
        chain = [("full", O.build_shard_payload({t: (v, None) for t, v in vals.items()}, "full", None,
                                                bitwidth, sorted(ROWS))[0])]
        for k in range(2):
            sel = {t: np.unique(rng.integers(0, r, max(1, r // 4))) for t, r in ROWS.items()}
            for t in ROWS:
                vals[t] = vals[t] + np.float32(0.5)
            chain.append(("incremental", O.build_shard_payload(
                {t: (v, None) for t, v in vals.items()}, "incremental", sel, bitwidth, sorted(ROWS))[0]))
        want = {t: np.zeros((r, dim), np.float32) for t, r in ROWS.items()}
        bits = {t: np.zeros((r + 7) // 8, np.uint8) for t, r in ROWS.items()}
        for kind, blob in chain:
            inc = kind == "incremental"
            for tid, sec in O.split_sections(blob, inc):
                O.apply_section(sec, inc, want[tid], None, bits[tid] if inc else None)
        out = {t.table_id: ds.DeviceTable(t.table_id, torch.zeros_like(t.values), row_base=t.row_base,
                                          total_rows=t.total_rows) for t in tables}
        tr = ds.ModelTracker({t: o.rows for t, o in out.items()}, device=dev)
        up = 0
        for kind, blob in chain:
            inc = kind == "incremental"
            apply_payload(blob, inc, out, {t: tr.baseline_bitmap(t) for t in out} if inc else None,
                          device=dev)
            up += apply_payload.last_h2d_bytes
        torch.cuda.synchronize()
        for t, o in out.items():
            lo, hi = o.row_base, o.row_base + o.rows
            if not np.array_equal(o.values.cpu().numpy().view(np.uint32), want[t][lo:hi].view(np.uint32)):
                ok = False
                print(f"RESTORE MISMATCH rank {rank} table {t}", flush=True)
            rb = np.unpackbits(bits[t], bitorder="little")[:ROWS[t]][lo:hi]
            gb = np.unpackbits(tr.baseline_bitmap(t).to_bytes(), bitorder="little")[:hi - lo]
            if not np.array_equal(rb, gb):
                ok = False
                print(f"BASELINE MISMATCH rank {rank} table {t}", flush=True)
        total = sum(len(b) for _, b in chain)
        if up > total * (1.0 / world + 0.05):
            ok = False
            print(f"rank {rank} uploaded {up} of {total} chain bytes", flush=True)
        oks = [None] * world
        dist.all_gather_object(oks, ok)
        ok = all(oks)
    if rank == 0 and ok:
        print("OK", flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
