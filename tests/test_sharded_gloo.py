"""Row-sharded checkpoint layout over a world_size-2 gloo group (CPU).

The multi-GPU path (paper_2010_08679_b200/sharded.py) splits
every table into contiguous row ranges; each rank writes the records of its
rows and the only exchange is the all_gather of per-table counts.  Here each
rank's records come from the oracle (the GPU writer is checked against the
oracle in test_gpu_parity.py), the counts go through a real gloo all_gather,
and rank 0 assembles the shard with the package's layout functions.  The
result must be byte-identical to the single-process payload of the whole
tables (engine.py:118-189).
"""
import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

ROWS = {0: 5000, 3: 777, 4: 1, 7: 12_345}
DIM = 16


class _T:
    def __init__(self, tid):
        self.table_id, self.dim = tid, DIM


def _tables():
    rng = np.random.default_rng(5)
    vals = {t: rng.standard_normal((r, DIM)).astype(np.float32) for t, r in ROWS.items()}
    sel = {t: np.sort(rng.choice(r, size=max(1, r // 7), replace=False)).astype(np.int64)
           for t, r in ROWS.items()}
    sel[4] = np.zeros(0, np.int64)  # a table with no dirty rows still has a header
    return vals, sel


def _worker(rank, world, port, kind, bitwidth, q):
    try:
        sys.path.insert(0, ROOT)
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from oracle import oracle as O
        from paper_2010_08679_b200.sharded import (assemble_shard, gather_counts, section_headers,
                                                   shard_layout, shard_rows)
        vals, sel = _tables()
        tids = sorted(ROWS)
        # the reference's DEFAULT_ADAPTIVE (quant.py:141-157) for 2/3/4 bits
        acfg = {2: (25, 0.5), 3: (25, 0.2), 4: (45, 0.2)}.get(bitwidth)
        runs, counts = [], []
        for t in tids:
            lo, hi = shard_rows(ROWS[t], world, rank)
            if kind == "incremental":
                mine = sel[t][(sel[t] >= lo) & (sel[t] < hi)]
                blob, _, _ = O.build_section(t, vals[t], mine, bitwidth=bitwidth, adaptive=acfg)
                counts.append(mine.size)
            else:
                blob, _, _ = O.build_section(t, vals[t][lo:hi], None, bitwidth=bitwidth,
                                             adaptive=acfg)
                counts.append(hi - lo)
            runs.append(blob[24:])  # records only: headers come from the global counts
        cnt = torch.tensor(counts + [sum(counts)], dtype=torch.int64)
        all_counts = gather_counts(cnt, world).view(world, -1)[:, :len(tids)].numpy()
        assert all_counts[rank].tolist() == counts
        rec = O.record_size(DIM, bitwidth, False, kind == "incremental")
        per_table, sec_off, run_off = shard_layout(all_counts, rank, rec)
        my_run = b"".join(runs)
        gathered = [None] * world
        dist.all_gather_object(gathered, my_run)
        if rank == 0:
            blob = assemble_shard(section_headers([_T(t) for t in tids], per_table, bitwidth),
                                  gathered, all_counts, rec)
            # this rank's runs sit at run_off in the assembled payload
            for g in range(world):
                pt, so, ro = shard_layout(all_counts, g, rec)
                off = 0
                for k in range(len(tids)):
                    n = int(all_counts[g, k]) * rec
                    assert blob[ro[k]:ro[k] + n] == gathered[g][off:off + n]
                    off += n
            assert len(blob) == sec_off[-1]
            whole = {t: (vals[t], None) for t in tids}
            ref, _, _ = O.build_shard_payload(whole, kind, sel if kind == "incremental" else None,
                                              bitwidth, tids)
            q.put(blob == ref)
        dist.barrier()
        dist.destroy_process_group()
    except Exception as e:  # surfaced by the parent
        q.put(repr(e))
        raise


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("kind,bitwidth", [("incremental", 8), ("incremental", 4),
                                           ("full", 8), ("incremental", None), ("full", 2)])
def test_row_sharded_shard_assembles_to_reference_bytes(kind, bitwidth):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    world, port = 2, _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, kind, bitwidth, q))
             for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
    res = q.get(timeout=5)
    assert res is True, res
    assert all(p.exitcode == 0 for p in procs)


def test_shard_layout_offsets():
    from paper_2010_08679_b200.sharded import shard_layout, shard_rows
    counts = np.array([[3, 0, 5], [2, 4, 0], [1, 1, 1]])
    rec = 32
    per_table, sec_off, run_off = shard_layout(counts, 1, rec)
    assert per_table.tolist() == [6, 5, 6]
    assert sec_off.tolist() == [0, 24 + 6 * 32, 48 + 11 * 32, 72 + 17 * 32]
    assert run_off.tolist() == [24 + 3 * 32, sec_off[1] + 24 + 0, sec_off[2] + 24 + 5 * 32]
    assert [shard_rows(10, 3, g) for g in range(3)] == [(0, 3), (3, 6), (6, 10)]
