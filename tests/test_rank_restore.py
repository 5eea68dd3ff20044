"""Rank-local restore slicing (engine.rank_slices, SURVEY 8(e) "Restore") on CPU:
each rank uploads only the records of its row range -- a slice of full
sections, a binary search over the sorted u64 row column of incremental
ones -- and the ranks together cover every record exactly once.  A
world_size-2 gloo group checks the cover across real processes."""

import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ROWS = {0: 5000, 3: 777, 4: 1, 7: 12_345}
DIM = 16


def _payload(kind, bitwidth, seed=5):
    rng = np.random.default_rng(seed)
    vals = {t: rng.standard_normal((r, DIM)).astype(np.float32) for t, r in ROWS.items()}
    sel = {t: np.sort(rng.choice(r, size=max(1, r // 7), replace=False)).astype(np.int64)
           for t, r in ROWS.items()}
    sel[4] = np.zeros(0, np.int64)
    blob, _, _ = O.build_shard_payload({t: (v, None) for t, v in vals.items()}, kind,
                                       sel if kind == "incremental" else None, bitwidth,
                                       sorted(ROWS), adaptive={4: (1, 0.5)})
    return blob, sel


def _records_of_rank(blob, kind, world, rank):
    """[(table, global row, record bytes)] a rank's slices address the way
    ds_restore_payload does (records [max(lo,0), min(hi,n)) of a full section
    through the biased offset; every sliced record of an incremental one)."""
    from paper_2010_08679_b200.engine import rank_slices
    from paper_2010_08679_b200.payload import parse_headers
    from paper_2010_08679_b200.sharded import shard_rows
    inc = kind == "incremental"
    infos = parse_headers(blob, inc)
    ranges = [shard_rows(ROWS[i.table_id], world, rank) for i in infos]
    host, descs = rank_slices(blob, infos, inc, ranges)
    out = []
    for info, (lo, hi), (off, n) in zip(infos, ranges, descs):
        rec = info.record_size
        if inc:
            for k in range(n):
                r = host[off + k * rec: off + (k + 1) * rec].tobytes()
                out.append((info.table_id, int.from_bytes(r[:8], "little"), r))
        else:
            for row in range(max(lo, 0), min(hi, info.rows)):
                out.append((info.table_id, row, host[off + row * rec: off + (row + 1) * rec].tobytes()))
    return out, host.size


def _all_records(blob, kind):
    from paper_2010_08679_b200.payload import parse_headers
    inc = kind == "incremental"
    buf = np.frombuffer(blob, np.uint8)
    out = []
    for info in parse_headers(blob, inc):
        rec = info.record_size
        for k in range(info.rows):
            r = buf[info.body_offset + k * rec: info.body_offset + (k + 1) * rec].tobytes()
            out.append((info.table_id, int.from_bytes(r[:8], "little") if inc else k, r))
    return out


@pytest.mark.parametrize("kind,bitwidth", [("incremental", 8), ("incremental", 4), ("full", 8),
                                           ("full", None), ("incremental", None)])
@pytest.mark.parametrize("world", (2, 3, 8))
def test_rank_slices_cover_every_record_once(kind, bitwidth, world):
    blob, _ = _payload(kind, bitwidth)
    got, nbytes = [], 0
    for rank in range(world):
        recs, n = _records_of_rank(blob, kind, world, rank)
        nbytes += n - 16
        from paper_2010_08679_b200.sharded import shard_rows
        for tid, row, _ in recs:
            lo, hi = shard_rows(ROWS[tid], world, rank)
            assert lo <= row < hi
        got += recs
    want = _all_records(blob, kind)
    assert sorted(got) == sorted(want)
    # the ranks together upload the record bytes once (headers stay on the host)
    assert nbytes == len(blob) - 24 * len(ROWS)


def test_rank_slices_unsorted_or_out_of_range_section_goes_whole():
    from paper_2010_08679_b200.engine import rank_slices
    from paper_2010_08679_b200.payload import parse_headers
    blob, _ = _payload("incremental", 8)
    infos = parse_headers(blob, True)
    bad = bytearray(blob)
    i0 = infos[0]
    bad[i0.body_offset: i0.body_offset + 8] = (10 ** 9).to_bytes(8, "little")  # id out of order/range
    host, descs = rank_slices(bytes(bad), parse_headers(bytes(bad), True), True,
                              [(0, 10)] * len(infos))
    assert descs[0][1] == infos[0].rows  # whole section: the kernel flags it like the reference


def _worker(rank, world, port, kind, q):
    try:
        sys.path.insert(0, ROOT)
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        blob, _ = _payload(kind, 8)
        recs, n = _records_of_rank(blob, kind, world, rank)
        gathered = [None] * world
        dist.all_gather_object(gathered, (recs, n))
        if rank == 0:
            allr = [r for g in gathered for r in g[0]]
            ok = sorted(allr) == sorted(_all_records(blob, kind))
            ok = ok and sum(g[1] - 16 for g in gathered) == len(blob) - 24 * len(ROWS)
            q.put(ok)
        dist.barrier()
        dist.destroy_process_group()
    except Exception as e:
        q.put(repr(e))
        raise


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("kind", ("incremental", "full"))
def test_rank_local_restore_cover_gloo(kind):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    world, port = 2, _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, kind, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
    res = q.get(timeout=5)
    assert res is True, res
    assert all(p.exitcode == 0 for p in procs)
