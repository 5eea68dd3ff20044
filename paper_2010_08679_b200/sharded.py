"""Row-sharded checkpointing across the GPUs of one box.

Every table is split into contiguous row ranges, one per rank
(rank g holds [row_base_g, row_base_g + rows_g)).  Each rank tracks,
compacts, quantizes and packs its own rows with no payload data crossing
GPUs.  The only exchange is an all_gather of the per-(rank, table) dirty
counts (NCCL over NVLink, a few hundred bytes): it fixes where each rank's
records land inside the shard payload, because a CNR1 section is one header
followed by fixed-size records in ascending row order (payload.py:84-104), so
the concatenation of the ranks' runs in rank order IS the reference section.
On GPUs the counts go over NVLink peer memory inside the writer's launch
(PeerCounts: CTA 0 stores them into every peer's buffer, the last CTA reads
every rank's); the NCCL all_gather (gather_counts) remains for gloo groups
and DS_COUNTS_EXCHANGE=nccl.

ShardedCheckpointer.step() is the stall-window work of one checkpoint
interval (engine.py:272-281 + the writer of :339-345): K1 over the
interval's lookups, K2 capture + fold, the count exchange, K3.  Nothing
synchronises the host until fetch().
"""

from __future__ import annotations

import ctypes
import os

import numpy as np
import torch

from . import _lib
from .engine import DeviceTable, ShardWriter, adaptive_for
from .payload import HEADER_SIZE, pack_header
from .tracker import LookupStream, ModelTracker


class PeerCounts:
    """The count exchange over NVLink peer memory, run inside K3.

    Every rank owns one exchange buffer (ds_peer_alloc); the IPC handles are
    swapped once at construction (all_gather_object) and every peer's buffer
    is mapped here.  arg(out) is the ds_peer_exchange of the next epoch for
    ShardWriter.write: the writer's CTA 0 stores this rank's counts into
    every peer's slot, its last CTA waits (bounded by timeout_s) for every
    rank's and copies them to `out`.  include/deltasnap_cuda.h gives the
    protocol.
    """

    def __init__(self, n: int, world: int, rank: int, group=None, device=None,
                 timeout_s: float = 60.0):
        import torch.distributed as dist
        L = _lib.lib()
        if world > _lib.PEER_MAX:
            raise ValueError(f"peer count exchange: at most {_lib.PEER_MAX} ranks")
        self.n, self.world, self.rank = n, world, rank
        self.device = device
        size = L.ds_peer_buffer_size(world, n)
        own = ctypes.c_void_p()
        handle = (ctypes.c_uint8 * 64)()
        with torch.cuda.device(device):
            _lib.check(L.ds_peer_alloc(size, ctypes.byref(own), handle), "peer_alloc")
            self._own = own.value
            handles = [None] * world
            dist.all_gather_object(handles, bytes(handle), group=group)
            ptrs, self._opened = [], []
            for r, h in enumerate(handles):
                if r == rank:
                    ptrs.append(self._own)
                    continue
                p = ctypes.c_void_p()
                hb = (ctypes.c_uint8 * 64).from_buffer_copy(h)
                _lib.check(L.ds_peer_open(hb, ctypes.byref(p)), "peer_open")
                ptrs.append(p.value)
                self._opened.append(p.value)
        self.flags = torch.zeros(1, dtype=torch.int32, device=device)
        self._x = _lib.PeerExchange()
        for r, p in enumerate(ptrs):
            self._x.peers[r] = p
        self._x.flags = self.flags.data_ptr()
        self._x.timeout_ns = int(timeout_s * 1e9)
        self._x.world, self._x.rank, self._x.epoch = world, rank, 0

    @property
    def epoch(self) -> int:
        return self._x.epoch

    def arg(self, out: torch.Tensor):
        """ds_peer_exchange of the next epoch, the counts landing in out."""
        self._x.epoch += 1
        self._x.out = out.data_ptr()
        return self._x

    def check(self) -> None:
        fl = int(self.flags.item())
        if fl:
            self.flags.zero_()  # a later healthy exchange must not re-raise this one
        _lib.raise_flags(fl, "count exchange")

    def close(self) -> None:
        """Unmap the peers' buffers and free this rank's (every rank must be
        done with the exchange: callers barrier first)."""
        L = _lib.lib()
        with torch.cuda.device(self.device):
            for p in self._opened:
                L.ds_peer_close(p)
            self._opened = []
            if self._own:
                L.ds_peer_free(self._own)
                self._own = None


def _use_peer_exchange(device, world: int, group) -> bool:
    """The peer exchange needs CUDA tables, an NCCL group (one box) and
    DS_COUNTS_EXCHANGE != "nccl" (the collective, kept for A/B)."""
    if world <= 1 or device.type != "cuda":
        return False
    if os.environ.get("DS_COUNTS_EXCHANGE", "peer") == "nccl":
        return False
    import torch.distributed as dist
    return dist.is_initialized() and dist.get_backend(group) == "nccl"


class ShardedCheckpointer:
    """One rank's part of a row-sharded incremental checkpoint.

    With world_size > 1 on an NCCL group the constructor is collective (the
    ranks swap their count-exchange buffers, PeerCounts), and every rank must
    then run the same sequence of checkpoints."""

    def __init__(self, tables: list, bitwidth: int | None, *, adaptive_overrides: dict | None = None,
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
        # ranges as the reference engine picks them (engine.py:112-115): the
        # greedy search at 2/3/4 bits unless overridden, naive at 8
        adaptive = adaptive_for(bitwidth, adaptive_overrides) if bitwidth is not None else None
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
        self._peer = PeerCounts(self.nt + 1, world_size, rank, group, self.device) \
            if _use_peer_exchange(self.device, world_size, group) else None
        self._comm = torch.cuda.Stream(self.device) \
            if (world_size > 1 and self._peer is None) else None
        self._stage_buf = None
        self._side = None
        self._pending = None

    # -- the device-side step ---------------------------------------------------

    def mark(self, idx, seg_off=None, seg_tables=None) -> None:
        """K1 over a stream of lookups: a device LookupStream (packed, mixed
        widths) or an int32/int64 tensor split by seg_off (local row ids)."""
        if isinstance(idx, LookupStream):
            self.tracker.mark_packed(idx)
        else:
            self.tracker.mark_batch(idx, seg_off, seg_tables)

    def checkpoint(self, staged_rows: int = 0):
        """K2, then K3 overlapped with the count all_gather, asynchronous on the
        current stream.  Only the host-side assembly needs the global counts, so
        the collective runs on a side stream while the writer runs; the
        current stream joins it before returning (step time includes it).

        staged_rows > 0 (stall-window staging): the dirty
        rows are gathered into a staging buffer of that many rows on the
        current stream, and K3 runs from the copy on a side stream; the
        returned event marks the end of the stall -- training may update the
        tables once the current stream passes it.  fetch()/layout() wait for
        the side stream.  (A dirty count above staged_rows raises at fetch.)
        """
        self.wait()  # a staged writer still reading ids / counts of the last one
        fold = 1
        self.counts = self.tracker.capture_into(self.ids, None, fold=fold, scope=self.scope)
        if staged_rows > 0:
            return self._checkpoint_staged(staged_rows)
        self.write()

    def write(self, staged: torch.Tensor | None = None) -> None:
        """K3 over the captured ids, with the count exchange when N > 1: inside
        the writer's launch over NVLink peer memory (PeerCounts), or the NCCL
        all_gather on a side stream beside it (gloo groups,
        DS_COUNTS_EXCHANGE=nccl).  Every rank's counts are in all_counts once
        the current stream passes this call."""
        args = (self.payload, self.ids, self.counts[:self.nt], None)
        if self.world == 1:
            self.writer.write(*args, local_ids=True, staged=staged)
        elif self._peer is not None:
            self.writer.write(*args, local_ids=True, staged=staged,
                              exchange=self._peer.arg(self.all_counts))
        else:
            main = torch.cuda.current_stream(self.device)
            self._comm.wait_stream(main)
            with torch.cuda.stream(self._comm):
                gather_counts(self.counts, self.world, self.group, out=self.all_counts)
            self.writer.write(*args, local_ids=True, staged=staged)
            main.wait_stream(self._comm)

    def _checkpoint_staged(self, cap: int):
        main = torch.cuda.current_stream(self.device)
        if self._stage_buf is None or self._stage_buf.shape[0] < cap:
            self._stage_buf = torch.empty((cap, self.tables[0].dim), dtype=torch.float32,
                                          device=self.device)
            self._side = torch.cuda.Stream(self.device)
        self.writer.stage_rows(self.ids, self.counts, self._stage_buf[:cap])
        stall_end = torch.cuda.Event(enable_timing=True)
        stall_end.record(main)
        self._side.wait_event(stall_end)
        with torch.cuda.stream(self._side):
            self.write(staged=self._stage_buf[:cap])
        self._pending = self._side
        return stall_end

    def wait(self) -> None:
        """Join a staged checkpoint's side stream into the current stream."""
        if self._pending is not None:
            torch.cuda.current_stream(self.device).wait_stream(self._pending)
            self._pending = None

    def step(self, idx, seg_off=None, seg_tables=None) -> None:
        self.mark(idx, seg_off, seg_tables)
        self.checkpoint()

    # -- host side ----------------------------------------------------------------

    def layout(self):
        """(local payload bytes, per-table local counts, per-table totals,
        section offsets, this rank's run offsets) after a sync; see shard_layout."""
        self.wait()
        if self._peer is not None:
            self._peer.check()
        counts_all = self.all_counts.view(self.world, self.nt + 1).cpu().numpy() \
            if self.world > 1 else self.counts.view(1, self.nt + 1).cpu().numpy()
        per_table, sec_off, run_off = shard_layout(counts_all[:, :self.nt], self.rank, self.rec)
        nbytes = int(self.writer.sec_off[-1].item())
        return nbytes, counts_all[self.rank, :self.nt], per_table, sec_off, run_off

    def headers(self, per_table) -> list:
        return section_headers(self.tables, per_table, self.bitwidth)

    def fetch(self, out: torch.Tensor | None = None, stream=None):
        """D2H of this rank's bytes into pinned memory; raises flagged errors."""
        self.wait()
        _lib.raise_flags(int(self.writer.flags.item()), "checkpoint")
        nbytes = int(self.writer.sec_off[-1].item())
        if out is None:
            out = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
        out[:nbytes].copy_(self.payload[:nbytes], non_blocking=True)
        return out, nbytes

    def assemble(self, rank_bytes: list, per_table) -> bytes:
        """Whole shard payload from every rank's (bytes, local counts) (host, rank order)."""
        if self.world == 1:
            return bytes(rank_bytes[0][0])
        return assemble_shard(self.headers(per_table), [bytes(b[0]) for b in rank_bytes],
                              np.stack([np.asarray(b[1]) for b in rank_bytes]), self.rec)


# ---------------------------------------------------------------------------
# host-side layout of a row-sharded shard payload (device independent)
# ---------------------------------------------------------------------------

def shard_layout(counts_all, rank: int, rec: int):
    """Byte layout of one shard payload assembled from every rank's runs.

    counts_all: (world, T) records per (rank, table).  Section t is one
    24-byte header (payload.py:88-91) followed by the runs of ranks 0..N-1 in
    rank order -- rows are sharded contiguously, so the runs concatenate to
    the ascending row order of the reference section (payload.py:84-104).
    Returns (per-table totals, section offsets [T+1], this rank's run offsets [T]).
    """
    counts_all = np.asarray(counts_all, dtype=np.int64)
    per_table = counts_all.sum(axis=0)
    sec_off = np.concatenate([[0], np.cumsum(HEADER_SIZE + per_table * rec)]).astype(np.int64)
    before = counts_all[:rank].sum(axis=0)
    run_off = sec_off[:-1] + HEADER_SIZE + before * rec
    return per_table, sec_off, run_off


def section_headers(tables, per_table, bitwidth, aux: bool = False) -> list:
    """The 24-byte CNR1 headers of a row-sharded shard (global row counts)."""
    return [pack_header(t.table_id, int(n), t.dim, bitwidth, 1 if bitwidth else 0, aux)
            for t, n in zip(tables, per_table)]


def assemble_shard(headers: list, runs: list, counts_all, rec: int) -> bytes:
    """Shard payload from the headers and each rank's concatenated runs."""
    counts_all = np.asarray(counts_all, dtype=np.int64)
    world, nt = counts_all.shape
    parts, offs = [], [0] * world
    for t in range(nt):
        parts.append(headers[t])
        for g in range(world):
            n = int(counts_all[g, t]) * rec
            parts.append(runs[g][offs[g]:offs[g] + n])
            offs[g] += n
    for g in range(world):
        if offs[g] != len(runs[g]):
            raise ValueError(f"rank {g}: run bytes {len(runs[g])} != counted {offs[g]}")
    return b"".join(parts)


def gather_counts(counts: torch.Tensor, world: int, group=None,
                  out: torch.Tensor | None = None) -> torch.Tensor:
    """all_gather of every rank's int64 per-table counts (the only collective;
    NCCL on GPUs, gloo in the CPU tests)."""
    import torch.distributed as dist
    if out is None:
        out = torch.empty(world * counts.numel(), dtype=counts.dtype, device=counts.device)
    if counts.is_cuda:
        dist.all_gather_into_tensor(out, counts, group=group)
    else:
        parts = [torch.empty_like(counts) for _ in range(world)]
        dist.all_gather(parts, counts, group=group)
        out.copy_(torch.cat(parts))
    return out


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
