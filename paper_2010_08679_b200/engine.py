"""Checkpoint writer and restore on the GPU (the engine.py hot-path mirror).

* build_shard_payload: drop-in for deltasnap/engine.py:118-189.  Same
  arguments and return value (payload bytes, quantized row count, summed row
  L2 error); the whole chunk loop runs in one writer launch (ds_writer.cu).
* ShardWriter: the device-resident form the training loop uses -- tables,
  ids and counts stay in HBM, nothing synchronises until the payload is
  copied to pinned host memory.
* apply_payload / restore_chain / restore: the _restore_at scatter
  (engine.py:443-512) on device tables (ds_restore.cu); chain/manifest logic
  stays on the host.

Differences from the reference, all on inputs the reference mishandles:
NaN/Inf rows raise DataError in every quantized mode (the reference's naive
8-bit path casts NaN codes silently); negative plan row ids raise BoundsError
(numpy would wrap them); err_sum agrees with the reference to ~1e-15 relative
(its float64 sum order depends on chunk_rows, engine.py:171-173).
"""

from __future__ import annotations

import contextlib
import ctypes
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from ._device import device_of, to_device
from .errors import ConfigError, IntegrityError, ShapeError
from .payload import HEADER_SIZE, parse_headers, record_size
from .quant import VALID_BITWIDTHS, AdaptiveConfig, default_adaptive_config

FULL = "full"
INCREMENTAL = "incremental"


@dataclass
class DeviceTable:
    """An embedding table (or a row shard of one) resident in HBM.

    values: (rows, dim) float32 CUDA tensor; row_base is the global id of
    local row 0; total_rows the global row count of the table.
    """

    table_id: int
    values: torch.Tensor
    aux: torch.Tensor | None = None
    row_base: int = 0
    total_rows: int | None = None

    def __post_init__(self):
        if self.total_rows is None:
            self.total_rows = self.row_base + self.values.shape[0]

    @property
    def rows(self) -> int:
        return self.values.shape[0]

    @property
    def dim(self) -> int:
        return self.values.shape[1]


def _nullctx():
    return contextlib.nullcontext()


def adaptive_for(bitwidth: int, overrides) -> AdaptiveConfig | None:
    """engine.py:112-115"""
    if overrides and bitwidth in overrides:
        return overrides[bitwidth]
    return default_adaptive_config(bitwidth)


def _as_device_table(t, device) -> DeviceTable:
    if isinstance(t, DeviceTable):
        return t
    values = to_device(t.values, torch.float32, device)
    aux = None if getattr(t, "aux", None) is None else to_device(t.aux, torch.float32, device)
    return DeviceTable(int(t.table_id), values, aux)


class ShardWriter:
    """K3 for a fixed set of device tables sharing one dim (<= 64 per launch).

    write() is asynchronous on the current stream; finish() synchronises,
    raises flagged data errors and returns (payload_bytes, err_sum).
    """

    def __init__(self, tables: list, bitwidth: int | None, *, adaptive: AdaptiveConfig | None = None,
                 aux: bool | None = None, write_headers: bool = True, device=None,
                 stats: torch.Tensor | None = None):
        if not tables:
            raise ValueError("ShardWriter needs at least one table")
        if len(tables) > _lib.MAX_TABLES:
            raise ValueError("at most 64 tables per ShardWriter; split the shard")
        if bitwidth is not None and bitwidth not in VALID_BITWIDTHS:
            raise ConfigError(f"unsupported bitwidth {bitwidth}")
        self.device = device_of(device if device is not None else tables[0].values.device)
        self.tables = tables
        dims = {t.dim for t in tables}
        if len(dims) != 1:
            raise ShapeError("tables of one ShardWriter must share dim")
        self.dim = dims.pop()
        self.bitwidth = bitwidth
        self.aux = all(t.aux is not None for t in tables) if aux is None else aux
        self.adaptive = adaptive if bitwidth is not None else None
        self.L = _lib.lib()
        descs = (_lib.TableDesc * len(tables))()
        for k, t in enumerate(tables):
            if t.values.dtype != torch.float32 or not t.values.is_cuda:
                raise ValueError("DeviceTable.values must be a float32 CUDA tensor")
            if t.values.stride(1) != 1:
                raise ValueError("DeviceTable.values rows must be contiguous")
            descs[k].values = t.values.data_ptr()
            descs[k].aux = t.aux.data_ptr() if (self.aux and t.aux is not None) else None
            descs[k].ld = t.values.stride(0)
            descs[k].rows = t.rows
            descs[k].row_base = t.row_base
            descs[k].ids_off = 0
            descs[k].table_id = t.table_id
            descs[k].dim = t.dim
        self._descs = descs
        self.params = _lib.CkptParams()
        self.params.bitwidth = bitwidth or 0
        self.params.adaptive_bins = self.adaptive.num_bins if self.adaptive else 0
        self.params.adaptive_steps = self.adaptive.steps if self.adaptive else 0
        self.params.write_headers = int(write_headers)
        self.params.aux = int(self.aux)
        self.params.stats = None if stats is None else stats.data_ptr()
        self.write_headers = write_headers
        ws = int(self.L.ds_writer_workspace_size(len(tables), sum(t.rows for t in tables), self.dim))
        self._ws = torch.zeros(ws, dtype=torch.uint8, device=self.device)  # zero before first use
        self.sec_off = torch.zeros(len(tables) + 1, dtype=torch.int64, device=self.device)
        self.err = torch.zeros(1, dtype=torch.float64, device=self.device)
        self.flags = torch.zeros(1, dtype=torch.int32, device=self.device)

    def record_size(self, incremental: bool) -> int:
        return record_size(self.dim, 1 if self.bitwidth else 0, self.bitwidth, self.aux,
                           incremental)

    def payload_bytes(self, counts) -> int:
        rec = self.record_size(counts is not None)
        rows = counts if counts is not None else [t.rows for t in self.tables]
        hdr = HEADER_SIZE if self.write_headers else 0
        return int(sum(hdr + int(n) * rec for n in rows))

    def write(self, payload: torch.Tensor, ids: torch.Tensor | None = None,
              counts: torch.Tensor | None = None, ids_offsets=None, *, local_ids: bool = False,
              stream=None, staged: torch.Tensor | None = None, exchange=None) -> None:
        """Launch layout + writer (+ error reduction).

        Incremental when `ids` is given: ids concatenates every table's row
        ids (ascending per table) and counts is a device int64 tensor of
        per-table lengths.  ids_offsets gives each table's start on the host;
        None means "packed" -- the starts are the prefix sums of counts,
        computed on the device (capture's layout, no host sync).  local_ids:
        the ids are table-local rows (capture output) instead of global ids.
        exchange: a ctypes ds_peer_exchange (sharded.PeerCounts.arg) -- the
        row-sharded count exchange then runs inside this launch.
        """
        incremental = ids is not None
        self.params.incremental = int(incremental)
        self.params.ids_packed = int(incremental and ids_offsets is None)
        self.params.ids_local = int(local_ids)
        # rows gathered by stage_rows (packed id order) instead of the live tables
        self.params.staged = staged.data_ptr() if staged is not None else None
        self.params.staged_rows = int(staged.shape[0]) if staged is not None else 0
        self.params.exchange = ctypes.addressof(exchange) if exchange is not None else None
        if incremental and ids_offsets is not None:
            for k in range(len(self.tables)):
                self._descs[k].ids_off = int(ids_offsets[k])
        if staged is None:  # (stage_rows cleared the flags for a staged write)
            self.flags.zero_()
        _lib.check(self.L.ds_write_payload(
            ctypes.cast(self._descs, ctypes.c_void_p), len(self.tables), ctypes.byref(self.params),
            ids.data_ptr() if incremental else None,
            counts.data_ptr() if incremental else None, payload.data_ptr(), payload.numel(),
            self.sec_off.data_ptr(), self.err.data_ptr(), self.flags.data_ptr(),
            self._ws.data_ptr(), self._ws.numel(), _lib.stream_handle(stream)), "write_payload")

    def stage_rows(self, ids: torch.Tensor, counts: torch.Tensor, staged: torch.Tensor,
                   stream=None) -> None:
        """Gather the dirty rows (packed table-local ids, counts with the total
        at [ntables]) into staged [capacity, dim]."""
        with torch.cuda.stream(stream) if stream is not None else _nullctx():
            self.flags.zero_()
        _lib.check(self.L.ds_stage_rows(
            ctypes.cast(self._descs, ctypes.c_void_p), len(self.tables), ids.data_ptr(),
            counts.data_ptr(), staged.shape[0], staged.data_ptr(), self.flags.data_ptr(),
            _lib.stream_handle(stream)), "stage_rows")

    def finish(self) -> tuple:
        """Synchronise; raise flagged errors; (total payload bytes, err_sum)."""
        flags = int(self.flags.item())
        _lib.raise_flags(flags, "build_shard_payload")
        total = int(self.sec_off[-1].item())
        return total, float(self.err.item())


def _group_tables(tables: list) -> list:
    """Consecutive runs of <= 64 tables sharing a dim (sections stay in order)."""
    groups, cur = [], []
    for t in tables:
        if cur and (t.dim != cur[0].dim or len(cur) == _lib.MAX_TABLES):
            groups.append(cur)
            cur = []
        cur.append(t)
    if cur:
        groups.append(cur)
    return groups


def build_shard_payload(snap, plan, shard_id: int, chunk_rows: int = 1024,
                        adaptive_overrides: dict | None = None, *, device=None) -> tuple:
    """Serialize one shard of a snapshot under a plan (engine.py:118-189).

    snap: anything with shard_tables(shard_id) returning tables with
    table_id/values/aux (the reference's ModelSnapshot, or DeviceTable lists);
    host arrays are uploaded, CUDA tensors used in place.  chunk_rows only
    changes the reference's float64 summation order of err_sum; the bytes do
    not depend on it (tests/test_engine.py:123-143 upstream).
    """
    del chunk_rows
    dev = device_of(device)
    incremental = plan.kind == INCREMENTAL
    bitwidth = plan.bitwidth
    acfg = adaptive_for(bitwidth, adaptive_overrides) if bitwidth is not None else None
    tables = [_as_device_table(t, dev) for t in snap.shard_tables(shard_id)]
    if not tables:
        return b"", 0, 0.0
    parts = []
    q_rows = 0
    err_sum = 0.0
    for group in _group_tables(tables):
        writer = ShardWriter(group, bitwidth, adaptive=acfg, device=dev)
        if incremental:
            sels = []
            for t in group:
                sel = plan.rows.get(t.table_id)
                sels.append(to_device(np.zeros(0, np.int64) if sel is None else sel, torch.int64,
                                      dev).reshape(-1))
            counts_h = [int(s.numel()) for s in sels]
            offs = np.concatenate([[0], np.cumsum(counts_h)]).astype(np.int64)
            ids = torch.cat(sels) if sum(counts_h) else torch.zeros(1, dtype=torch.int64,
                                                                    device=dev)
            counts = torch.tensor(counts_h, dtype=torch.int64, device=dev)
            nbytes = writer.payload_bytes(counts_h)
            payload = torch.empty(nbytes + 16, dtype=torch.uint8, device=dev)
            writer.write(payload, ids, counts, offs[:-1])
            n_rows = sum(counts_h)
        else:
            nbytes = writer.payload_bytes(None)
            payload = torch.empty(nbytes + 16, dtype=torch.uint8, device=dev)
            writer.write(payload)
            n_rows = sum(t.rows for t in group)
        total, err = writer.finish()
        assert total == nbytes, (total, nbytes)
        parts.append(payload[:total].cpu().numpy().tobytes())
        if bitwidth is not None:
            q_rows += n_rows
            err_sum += err
    return b"".join(parts), q_rows, err_sum


# ---------------------------------------------------------------------------
# restore (engine.py:443-535)
# ---------------------------------------------------------------------------

def _upload_payload(data, dev) -> torch.Tensor:
    buf = np.frombuffer(data, dtype=np.uint8)
    out = torch.empty(buf.size + 16, dtype=torch.uint8, device=dev)
    if buf.size:
        host = torch.from_numpy(buf.copy()).pin_memory()
        out[:buf.size].copy_(host, non_blocking=True)
    return out


_DUMMY = {}


def _dummy_rows(dev) -> torch.Tensor:
    if dev not in _DUMMY:
        _DUMMY[dev] = torch.zeros(4, dtype=torch.float32, device=dev)
    return _DUMMY[dev]


def rank_slices(data, infos: list, incremental: bool, ranges: list):
    """The records of each section that fall in one rank's row range
    (SURVEY 8(e) "Restore": a slice for full sections, a binary search over
    the sorted u64 row column for incremental ones, engine.py:459-485).

    ranges: [(row_lo, row_hi)] per section.  Returns (host uint8 array of the
    concatenated slices + 16 bytes of slack, [(body_off, nrec)] per section)
    for ds_restore_payload against that array: a full section's body_off is
    biased by -row_lo records, so record i still addresses global row i.  A
    section whose row column is not strictly ascending or holds an id
    outside the table goes whole (the kernel then flags it exactly as the
    reference would fail it)."""
    buf = np.frombuffer(data, dtype=np.uint8)
    parts, descs, pos = [], [], 0
    for info, (lo, hi) in zip(infos, ranges):
        rec = info.record_size
        body = buf[info.body_offset: info.body_offset + info.rows * rec]
        if incremental:
            k0, k1 = 0, info.rows
            if info.rows:
                ids = body.reshape(info.rows, rec)[:, :8].copy().view("<i8").reshape(-1)
                ok = ids[0] >= 0 and bool(np.all(ids[1:] > ids[:-1]))
                if ok:
                    k0, k1 = (int(v) for v in np.searchsorted(ids, [lo, hi]))
            parts.append(body[k0 * rec: k1 * rec])
            descs.append((pos, k1 - k0))
            pos += (k1 - k0) * rec
        else:
            k0, k1 = max(0, min(lo, info.rows)), max(0, min(hi, info.rows))
            k1 = max(k0, k1)
            parts.append(body[k0 * rec: k1 * rec])
            descs.append((pos - k0 * rec, info.rows))
            pos += (k1 - k0) * rec
    parts.append(np.zeros(16, np.uint8))
    return np.concatenate(parts), descs


def apply_payload(data, incremental: bool, tables: dict, baseline: dict | None = None,
                  device=None, device_buf: torch.Tensor | None = None, sync: bool = True,
                  rank_local: bool | None = None, slice_descs: list | None = None):
    """Apply one shard payload to device tables (the loop body of
    engine.py:625-649).

    tables: {table_id: DeviceTable} (row shards allowed: only rows in
    [row_base, row_base+rows) are written); baseline: {table_id: DirtyBitmap}
    of the since-baseline scope rebuilt for incremental sections (:476).
    Errors are raised in the reference's order: the first failing section
    wins; within a section FormatError precedes IntegrityError.
    device_buf: the same bytes already in device memory (no upload);
    sync=False: launch only and return a callable that checks the flags later
    (restore pipelines check once per chain).  rank_local (default: the
    tables are row shards and the bytes are on the host): upload only the
    records of this rank's rows (rank_slices) instead of the whole payload.
    slice_descs: device_buf holds rank_slices' array, these its descriptors.
    """
    dev = device_of(device)
    infos = parse_headers(data, incremental)  # FormatError for any bad header
    if not infos:
        return (lambda: None) if not sync else None
    L = _lib.lib()
    flags = torch.zeros(len(infos), dtype=torch.int32, device=dev)
    # host-side checks first: sections from the first failing one on are not applied
    host_err = None
    for k, info in enumerate(infos):
        t = tables.get(info.table_id)
        if t is None:
            host_err = (k, IntegrityError(f"payload names unknown table {info.table_id}"))
        elif info.dim != t.dim:
            host_err = (k, IntegrityError(f"dim mismatch in table {info.table_id}"))
        elif not incremental and info.rows != t.total_rows:
            host_err = (k, IntegrityError(
                f"full section for table {info.table_id} has {info.rows} rows, "
                f"expected {t.total_rows}"))
        if host_err is not None:
            break
    napply = len(infos) if host_err is None else host_err[0]
    buf = device_buf
    body_off = [info.body_offset for info in infos]
    nrec = [info.rows for info in infos]
    if slice_descs is not None:
        for k, (o, n) in enumerate(slice_descs[:napply]):
            body_off[k], nrec[k] = o, n
        rank_local = False
    if rank_local is None:
        rank_local = device_buf is None and any(
            t.row_base > 0 or t.row_base + t.rows < t.total_rows for t in tables.values())
    if rank_local and device_buf is None and napply:
        ranges = [(tables[i.table_id].row_base, tables[i.table_id].row_base + tables[i.table_id].rows)
                  for i in infos[:napply]]
        host, descs = rank_slices(data, infos[:napply], incremental, ranges)
        buf = torch.empty(host.size, dtype=torch.uint8, device=dev)
        buf.copy_(torch.from_numpy(host).pin_memory(), non_blocking=True)
        for k, (o, n) in enumerate(descs):
            body_off[k], nrec[k] = o, n
        apply_payload.last_h2d_bytes = int(host.size)
    elif device_buf is None:
        buf = _upload_payload(data, dev)
        apply_payload.last_h2d_bytes = len(data)
    stream = _lib.stream_handle()
    # one launch per run of sections sharing (dim, bitwidth, aux) -- normally
    # the whole payload (ds_restore_payload, <= 64 sections per launch)
    k0 = 0
    while k0 < napply:
        key = (infos[k0].dim, infos[k0].bitwidth, infos[k0].aux)
        k1 = k0
        while (k1 < napply and k1 - k0 < _lib.MAX_TABLES and
               (infos[k1].dim, infos[k1].bitwidth, infos[k1].aux) == key):
            k1 += 1
        # ds_restore_sec rows (9 x 64-bit fields, include/deltasnap_cuda.h)
        secs = np.empty((k1 - k0, 9), dtype=np.int64)
        for j, info in enumerate(infos[k0:k1]):
            t = tables[info.table_id]
            bm = baseline.get(info.table_id) if (baseline is not None and incremental) else None
            # a rank may hold no rows of a table: any valid address (nothing is written)
            secs[j] = (body_off[k0 + j], nrec[k0 + j],
                       t.values.data_ptr() or _dummy_rows(dev).data_ptr(),
                       t.aux.data_ptr() if (info.aux and t.aux is not None) else 0,
                       0 if bm is None else bm.words.data_ptr(),
                       t.values.stride(0), t.total_rows, t.row_base, t.row_base + t.rows)
        _lib.check(L.ds_restore_payload(
            buf.data_ptr(), secs.ctypes.data, k1 - k0, key[0], key[1] or 0,
            int(key[2]), int(incremental), flags[k0:].data_ptr(), stream), "restore_payload")
        k0 = k1

    def check():
        fl = flags.cpu().numpy()
        first_dev = next((k for k in range(len(infos)) if fl[k]), None)
        if first_dev is not None and (host_err is None or first_dev < host_err[0]):
            _lib.raise_flags(int(fl[first_dev]), f"restore (table {infos[first_dev].table_id})")
        if host_err is not None:
            raise host_err[1]

    if not sync:
        return check
    check()


@dataclass
class RestoredTables:
    """What restore produces on the GPU: device tables + rebuilt tracker."""

    tables: dict
    tracker: object
    chain_ids: list = field(default_factory=list)
    manifest: object = None
    dense: np.ndarray | None = None


def restore_chain(chain: list, table_shapes: dict, *, aux: bool = False, device=None,
                  row_range: tuple | None = None) -> RestoredTables:
    """Rebuild tables from a manifest chain (engine.py:443-512 scatter part).

    chain: [(kind, [shard payload bytes, ...]), ...] in chain order (base
    first; later entries override earlier ones); table_shapes: {tid: (rows,
    dim)}; row_range=(lo, hi) restores only that global row range of every
    table (one rank of a row-sharded restore).
    """
    from .tracker import ModelTracker

    dev = device_of(device)
    tables = {}
    for tid, (rows, dim) in sorted(table_shapes.items()):
        lo, hi = (0, rows) if row_range is None else (max(0, row_range[0]), min(rows, row_range[1]))
        n = max(0, hi - lo)
        tables[tid] = DeviceTable(tid, torch.zeros((n, dim), dtype=torch.float32, device=dev),
                                  torch.zeros((n, dim), dtype=torch.float32, device=dev)
                                  if aux else None, row_base=lo, total_rows=rows)
    tracker = ModelTracker({tid: t.rows for tid, t in tables.items()}, device=dev)
    baseline = {tid: tracker.baseline_bitmap(tid) for tid in tables}
    for kind, payloads in chain:
        inc = kind == INCREMENTAL
        for data in payloads:
            # (host bytes, device copy) pairs come from stage_chain
            host, dbuf = data if isinstance(data, tuple) else (data, None)
            apply_payload(host, inc, tables, baseline if inc else None, device=dev, device_buf=dbuf)
    return RestoredTables(tables=tables, tracker=tracker)


def stage_chain(chain: list, checksums: list | None = None, device=None) -> list:
    """Move a chain's payloads to the device and verify them there before
    anything is applied (store.py:488-507 verify).

    chain: [(kind, [payload bytes, ...]), ...]; checksums: matching
    [[crc32, ...], ...] (manifest ObjectEntry.crc32) or None.  Each payload
    is H2D-copied from pinned memory on a copy stream while the previous one
    is checksummed on the device (ds_crc32); one sync at the end compares
    every CRC and raises IntegrityError for the first mismatch, like the
    reference.  Returns the chain with (bytes, device buffer) pairs for
    restore_chain.
    """
    from .payload import crc32 as dev_crc32

    dev = device_of(device)
    main = torch.cuda.current_stream(dev)
    copy = torch.cuda.Stream(dev)
    staged, crcs, want = [], [], []
    for ci, (kind, payloads) in enumerate(chain):
        out = []
        for pi, data in enumerate(payloads):
            buf = np.frombuffer(data, dtype=np.uint8)
            dbuf = torch.empty(buf.size + 16, dtype=torch.uint8, device=dev)
            if buf.size:
                host = torch.from_numpy(buf.copy()).pin_memory()
                with torch.cuda.stream(copy):
                    dbuf[:buf.size].copy_(host, non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(copy)
                main.wait_event(ev)  # the CRC of this payload runs after its copy
            if checksums is not None:
                c = torch.zeros(1, dtype=torch.int32, device=dev)
                dev_crc32(dbuf, buf.size, out=c)
                crcs.append(c)
                want.append((checksums[ci][pi], f"payload {pi} of chain entry {ci}"))
            out.append((data, dbuf))
        staged.append((kind, out))
    if crcs:
        got = torch.cat(crcs).cpu().numpy().astype(np.uint32)
        for g, (w, what) in zip(got, want):
            if int(g) != (int(w) & 0xFFFFFFFF):
                raise IntegrityError(f"checksum mismatch for {what}")
    return staged


# ---------------------------------------------------------------------------
# what restore() returns: the reference's RestoredRun (engine.py:415-425) with
# the tables resident in HBM
# ---------------------------------------------------------------------------

@dataclass
class DeviceModelConfig:
    """ModelConfig (model.py:18-40) as config_from_manifest (engine.py:427-440)
    derives it.  The reference raises IntegrityError for mixed table shapes;
    the device restore allows them (Criteo-shaped tables): rows_per_table and
    dim are then None and `shapes` holds every table's (rows, dim)."""

    num_tables: int
    rows_per_table: int | None
    dim: int | None
    num_shards: int = 1
    has_aux_state: bool = False
    dense_dim: int = 256
    shapes: dict = field(default_factory=dict)

    def validate(self) -> None:
        """model.py:27-37 (ConfigError), per table for mixed shapes."""
        if self.num_tables < 1:
            raise ConfigError("num_tables must be >= 1")
        if any(r < 1 for r, _ in self.shapes.values()):
            raise ConfigError("rows_per_table must be >= 1")
        if any(d < 1 for _, d in self.shapes.values()):
            raise ConfigError("dim must be >= 1")
        if self.num_shards < 1:
            raise ConfigError("num_shards must be >= 1")
        if self.dense_dim < 1:
            raise ConfigError("dense_dim must be >= 1")

    def shard_of(self, table_id: int) -> int:
        return table_id % self.num_shards  # model.py:39-40


@dataclass
class ReaderPosition:
    """ReaderState (model.py:67-80)."""

    batches_consumed: int = 0
    rng_cursor: int = 0

    def copy(self) -> "ReaderPosition":
        return ReaderPosition(self.batches_consumed, self.rng_cursor)


@dataclass
class DeviceModelState:
    """ModelState (model.py:83-98) with DeviceTable tables.  shard_tables()
    has the reference's meaning, so a restored model feeds
    build_shard_payload directly."""

    config: DeviceModelConfig
    tables: dict
    dense: np.ndarray
    reader: ReaderPosition = field(default_factory=ReaderPosition)

    def shard_tables(self, shard_id: int) -> list:
        return [t for tid, t in sorted(self.tables.items())
                if self.config.shard_of(tid) == shard_id]

    def host_tables(self) -> dict:
        """{tid: (values, aux | None)} as float32 numpy arrays (D2H)."""
        return {tid: (t.values.cpu().numpy(), None if t.aux is None else t.aux.cpu().numpy())
                for tid, t in sorted(self.tables.items())}


@dataclass
class IntervalSizes:
    """IntervalHistory (policy.py:23-44): increment sizes as fractions of the
    baseline's bytes, clamped to 1.0."""

    sizes: list = field(default_factory=list)

    def record(self, fraction: float) -> None:
        import math

        from .errors import DataError
        if not math.isfinite(fraction) or fraction < 0.0:
            raise DataError(f"invalid increment fraction {fraction!r}")
        self.sizes.append(min(fraction, 1.0))

    def reset(self) -> None:
        self.sizes.clear()

    def __len__(self) -> int:
        return len(self.sizes)


@dataclass
class RestoredRun:
    """Everything needed to resume training from a committed checkpoint
    (engine.py:415-425): same fields, tables in HBM, tracker on the device
    with the since-baseline scope rebuilt (engine.py:476)."""

    model: DeviceModelState
    tracker: object
    history: IntervalSizes
    baseline_id: int
    baseline_payload_bytes: int
    manifest: object
    chain_ids: list

    # pre-RestoredRun field names (restore_chain's RestoredTables)
    @property
    def tables(self) -> dict:
        return self.model.tables

    @property
    def dense(self) -> np.ndarray:
        return self.model.dense

    def to_reference(self, deltasnap, tracker: str = "device"):
        """The reference's own RestoredRun over host copies, for code that
        needs numpy tables (sim.apply_batch, state_digest): `deltasnap` is
        the reference package; tracker="device" keeps this tracker (a drop-in
        for deltasnap.tracker.ModelTracker), "reference" copies the rebuilt
        since-baseline bits into a reference ModelTracker."""
        M = deltasnap.model
        cfg = self.model.config
        if cfg.rows_per_table is None:
            raise IntegrityError("tables with mixed shapes are not supported")
        tables = {tid: M.EmbeddingTable(tid, v, a)
                  for tid, (v, a) in self.model.host_tables().items()}
        model = M.ModelState(
            config=M.ModelConfig(num_tables=cfg.num_tables, rows_per_table=cfg.rows_per_table,
                                 dim=cfg.dim, num_shards=cfg.num_shards,
                                 has_aux_state=cfg.has_aux_state, dense_dim=cfg.dense_dim),
            tables=tables, dense=self.model.dense.copy(),
            reader=M.ReaderState(self.model.reader.batches_consumed, self.model.reader.rng_cursor))
        tr = self.tracker
        if tracker == "reference":
            tr = deltasnap.tracker.ModelTracker({tid: t.rows for tid, t in tables.items()})
            for tid in tables:
                tr.mark_baseline(tid, self.tracker.baseline_bitmap(tid).dirty_rows()[0])
        hist = deltasnap.policy.IntervalHistory()
        hist.sizes.extend(self.history.sizes)
        return deltasnap.engine.RestoredRun(
            model=model, tracker=tr, history=hist, baseline_id=self.baseline_id,
            baseline_payload_bytes=self.baseline_payload_bytes, manifest=self.manifest,
            chain_ids=list(self.chain_ids))


def state_digest(state) -> str:
    """model.py:156-165: SHA-256 over every table (values, then aux) in table
    order, then the dense vector -- for device or host models."""
    import hashlib
    h = hashlib.sha256()
    for tid in sorted(state.tables):
        t = state.tables[tid]
        for a in (t.values, t.aux):
            if a is None:
                continue
            a = a.cpu().numpy() if isinstance(a, torch.Tensor) else a
            h.update(np.ascontiguousarray(a).tobytes())
    dense = state.dense.cpu().numpy() if isinstance(state.dense, torch.Tensor) else state.dense
    h.update(np.ascontiguousarray(dense).tobytes())
    return h.hexdigest()


def _dense_from_bytes(data: bytes, dense_dim: int) -> np.ndarray:
    """engine.py:196-199"""
    from .errors import FormatError
    if len(data) != dense_dim * 4:
        raise FormatError(f"dense payload has {len(data)} bytes, expected {dense_dim * 4}")
    return np.frombuffer(data, dtype="<f4").astype(np.float32)


def _config_from_manifest(target) -> DeviceModelConfig:
    """engine.py:427-440, mixed shapes allowed (see DeviceModelConfig)."""
    shapes = {tid: (int(info.rows), int(info.dim)) for tid, info in target.tables.items()}
    rows = {r for r, _ in shapes.values()}
    dims = {d for _, d in shapes.values()}
    return DeviceModelConfig(
        num_tables=len(shapes),
        rows_per_table=rows.pop() if len(rows) == 1 else None,
        dim=dims.pop() if len(dims) == 1 else None,
        num_shards=len(target.shards), has_aux_state=bool(target.aux),
        dense_dim=target.dense.nbytes // 4, shapes=shapes)


def _verify_presence(cstore, chain) -> None:
    """store.verify (store.py:488-501) minus the shard checksums, which
    stage_chain checks on the device: presence and size of every object, and
    the dense objects' CRC32 on the host (a few KB)."""
    import zlib
    for m in chain:
        for e in list(m.shards.values()) + [m.dense]:
            try:
                data = cstore.store.get(e.key)
            except KeyError:
                raise IntegrityError(f"missing object {e.key!r}") from None
            if len(data) != e.nbytes:
                raise IntegrityError(f"size mismatch for {e.key!r}: {len(data)} != {e.nbytes}")
            if e is m.dense and (zlib.crc32(data) & 0xFFFFFFFF) != (int(e.crc32) & 0xFFFFFFFF):
                raise IntegrityError(f"checksum mismatch for {e.key!r}")


def _restore_at(cstore, ckpt_id: int, device=None, verify_on_device: bool = False,
                row_range: tuple | None = None) -> RestoredRun:
    """engine.py:443-512 with the decode + scatter on the GPU."""
    if verify_on_device:
        chain = cstore.resolve_chain(ckpt_id)
        _verify_presence(cstore, chain)
    else:
        chain = cstore.verify_chain(ckpt_id)
    base, target = chain[0], chain[-1]
    config = _config_from_manifest(target)
    config.validate()
    plan = [(m.kind, [cstore.store.get(e.key) for _, e in sorted(m.shards.items())])
            for m in chain]
    if verify_on_device:
        sums = [[e.crc32 for _, e in sorted(m.shards.items())] for m in chain]
        plan = stage_chain(plan, sums, device=device)
    out = restore_chain(plan, config.shapes, aux=bool(target.aux), device=device,
                        row_range=row_range)
    dense = _dense_from_bytes(cstore.store.get(target.dense.key), config.dense_dim)
    model = DeviceModelState(config=config, tables=out.tables, dense=dense,
                             reader=ReaderPosition(target.reader_batches, target.reader_cursor))
    # engine.py:495-502
    history = IntervalSizes()
    if base.payload_bytes > 0:
        for mid in cstore.valid_ids():
            if mid <= base.checkpoint_id or mid > target.checkpoint_id:
                continue
            m = cstore.read_manifest(mid)
            if m.kind == INCREMENTAL and m.base_id == base.checkpoint_id:
                history.record(m.payload_bytes / base.payload_bytes)
    return RestoredRun(model=model, tracker=out.tracker, history=history,
                       baseline_id=base.checkpoint_id,
                       baseline_payload_bytes=base.payload_bytes, manifest=target,
                       chain_ids=[m.checkpoint_id for m in chain])


def _restore_errors():
    """(IntegrityError, FormatError) of this package and, when the caller's
    store raises the reference package's own classes, of that package too."""
    from . import errors
    out = [errors.IntegrityError, errors.FormatError]
    import sys
    ref = sys.modules.get("deltasnap.errors")
    if ref is not None:
        out += [ref.IntegrityError, ref.FormatError]
    return tuple(out)


def restore(cstore, *, fallback: bool = False, checkpoint_id: int | None = None,
            device=None, verify_on_device: bool = False,
            row_range: tuple | None = None) -> RestoredRun:
    """Rebuild the model from the newest valid checkpoint (engine.py:515-535).

    cstore: the reference's CheckpointStore (or anything with its
    resolve_chain / verify_chain / valid_ids / read_manifest / store.get).
    Chain resolution stays on the host; decode and scatter run on the GPU.
    verify_on_device: the shard payloads' CRC32 checks of store.verify run on
    the device after the H2D copy (stage_chain); presence, sizes and the dense
    objects' CRC32 are checked on the host.  row_range=(lo, hi): restore only
    that global row range of every table (one rank of a row-sharded restore).
    With fallback=True a checkpoint failing integrity checks is skipped and
    the next older one tried.
    """
    kw = dict(device=device, verify_on_device=verify_on_device, row_range=row_range)
    if checkpoint_id is not None:
        return _restore_at(cstore, checkpoint_id, **kw)
    ids = cstore.valid_ids()
    if not ids:
        raise IntegrityError("no valid checkpoint to restore from")
    caught = _restore_errors()
    last = None
    for cid in reversed(ids):
        try:
            return _restore_at(cstore, cid, **kw)
        except caught as exc:
            if not fallback:
                raise
            last = exc
    raise IntegrityError(f"no restorable checkpoint: {last}")
