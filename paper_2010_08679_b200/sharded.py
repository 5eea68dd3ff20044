"""Row-sharded checkpointing across the GPUs of one box.

Every table is split into contiguous row ranges, one per rank
(rank g holds [row_base_g, row_base_g + rows_g)).  Each rank tracks,
compacts, quantizes and packs its own rows with no payload data crossing
GPUs.  The only exchange is an all_gather of the per-(rank, table) dirty
counts (NCCL over NVLink, a few hundred bytes): it fixes where each rank's
records land inside the shard payload, because a CNR1 section is one header
followed by fixed-size records in ascending row order (payload.py:84-104), so
the concatenation of the ranks' runs in rank order IS the reference section.

ShardedCheckpointer.step() is the stall-window work of one checkpoint
interval (engine.py:272-281 + the writer of :339-345): K1 over the
interval's lookups, K2 capture + fold, the count all_gather, K3.  Nothing
synchronises the host until fetch().
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib
from .engine import DeviceTable, ShardWriter
from .payload import HEADER_SIZE, pack_header
from .quant import AdaptiveConfig
from .tracker import ModelTracker


class ShardedCheckpointer:
    """One rank's part of a row-sharded incremental checkpoint."""

    def __init__(self, tables: list, bitwidth: int | None, *, adaptive: AdaptiveConfig | None = None,
                 rank: int = 0, world_size: int = 1, group=None, device=None,
                 scope: str = "interval"):
        self.tables = tables
        self.device = tables[0].values.device if device is None else torch.device(device)
        self.rank, self.world = rank, world_size
        self.group = group
        self.scope = scope
        self.nt = len(tables)
        self.bitwidth = bitwidth
        self.tracker = ModelTracker({t.table_id: t.rows for t in tables}, device=self.device)
        # one rank writes whole sections (headers included); with several
        # ranks the runs are written bare and headers come from the counts
        self.writer = ShardWriter(tables, bitwidth, adaptive=adaptive, device=self.device,
                                  write_headers=(world_size == 1))
        self.rec = self.writer.record_size(True)
        total_rows = sum(t.rows for t in tables)
        self.ids = torch.empty(max(1, total_rows), dtype=torch.int64, device=self.device)
        self.counts = torch.zeros(self.nt + 1, dtype=torch.int64, device=self.device)
        self.all_counts = torch.zeros(world_size * (self.nt + 1), dtype=torch.int64,
                                      device=self.device)
        hdr = HEADER_SIZE if world_size == 1 else 0
        self.capacity = sum(hdr + t.rows * self.rec for t in tables)
        self.payload = torch.empty(self.capacity + 16, dtype=torch.uint8, device=self.device)
        self._seg_cache = None

    # -- the device-side step ---------------------------------------------------

    def mark(self, idx: torch.Tensor, seg_off, seg_tables) -> None:
        """K1 over a stream of lookups (int32 or int64 local row ids)."""
        self.tracker.mark_batch(idx, seg_off, seg_tables)

    def checkpoint(self) -> None:
        """K2 + count all_gather + K3, asynchronous on the current stream."""
        fold = 1
        self.tracker.capture_into(self.ids, self.counts, fold=fold, scope=self.scope)
        if self.world > 1:
            import torch.distributed as dist
            dist.all_gather_into_tensor(self.all_counts, self.counts, group=self.group)
        self.writer.write(self.payload, self.ids, self.counts[:self.nt], None, local_ids=True)

    def step(self, idx: torch.Tensor, seg_off, seg_tables) -> None:
        self.mark(idx, seg_off, seg_tables)
        self.checkpoint()

    # -- host side ----------------------------------------------------------------

    def layout(self):
        """(local payload bytes, per-table local counts, global offsets) after a sync.

        Global layout of the shard payload: section t = header (24 B) + the
        runs of ranks 0..N-1; this rank's run of table t starts at
        run_off[t] (bytes from the payload start).
        """
        counts_all = self.all_counts.view(self.world, self.nt + 1).cpu().numpy() \
            if self.world > 1 else self.counts.view(1, self.nt + 1).cpu().numpy()
        local = counts_all[self.rank, :self.nt]
        per_table = counts_all[:, :self.nt].sum(axis=0)
        sec_off = np.concatenate([[0], np.cumsum(HEADER_SIZE + per_table * self.rec)])
        before = counts_all[:self.rank, :self.nt].sum(axis=0)
        run_off = sec_off[:-1] + HEADER_SIZE + before * self.rec
        nbytes = int(self.writer.sec_off[-1].item())
        return nbytes, local, per_table, sec_off, run_off

    def headers(self, per_table) -> list:
        return [pack_header(t.table_id, int(n), t.dim, self.bitwidth, 1 if self.bitwidth else 0,
                            False) for t, n in zip(self.tables, per_table)]

    def fetch(self, out: torch.Tensor | None = None, stream=None):
        """D2H of this rank's bytes into pinned memory; raises flagged errors."""
        _lib.raise_flags(int(self.writer.flags.item()), "checkpoint")
        nbytes = int(self.writer.sec_off[-1].item())
        if out is None:
            out = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
        out[:nbytes].copy_(self.payload[:nbytes], non_blocking=True)
        return out, nbytes

    def assemble(self, rank_bytes: list, per_table) -> bytes:
        """Whole shard payload from every rank's fetched runs (host, rank order)."""
        if self.world == 1:
            return bytes(rank_bytes[0])
        parts = []
        offs = [0] * self.world
        counts = [None] * self.world
        for g in range(self.world):
            counts[g] = rank_bytes[g][1]
        for t, hdr in enumerate(self.headers(per_table)):
            parts.append(hdr)
            for g in range(self.world):
                n = int(counts[g][t]) * self.rec
                parts.append(bytes(rank_bytes[g][0][offs[g]:offs[g] + n]))
                offs[g] += n
        return b"".join(parts)


def shard_rows(rows: int, world: int, rank: int) -> tuple:
    """Contiguous row range [lo, hi) of `rank`."""
    lo = rows * rank // world
    hi = rows * (rank + 1) // world
    return lo, hi


def make_local_tables(shapes: dict, world: int, rank: int, device, init=None) -> list:
    """Row shards of every table for one rank, as DeviceTables."""
    out = []
    for tid, (rows, dim) in sorted(shapes.items()):
        lo, hi = shard_rows(rows, world, rank)
        values = torch.empty((hi - lo, dim), dtype=torch.float32, device=device)
        if init is not None:
            init(tid, lo, values)
        out.append(DeviceTable(tid, values, row_base=lo, total_rows=rows))
    return out
