"""Dirty-row tracking on the GPU (K0/K1/K2).

Mirror of deltasnap/tracker.py:19-139.  Bitmaps live in HBM as uint32 words
(bit r of a table at word r>>5, bit r&31), byte-identical to the reference's
uint8[(rows+7)//8] bitset; `nbytes` reports that logical size.  A
ModelTracker keeps every table's words in one buffer per scope so that
capture() compacts all tables with one three-kernel pass (ds_capture).

Error timing: host (numpy / list) indices are bounds-checked before the
upload, so BoundsError is raised by mark() itself with no bit set, exactly
like the reference (tracker.py:32-35).  Device-tensor indices are checked by
the kernel; the error is raised at the next synchronising call (capture,
dirty_rows, popcount, check()).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._device import check_flags, device_of, new_flags
from .errors import BoundsError, ShapeError


def _words_for(rows: int) -> int:
    return (rows + 31) // 32


def _host_ids(indices, rows: int, table_id: int) -> np.ndarray:
    idx = np.asarray(indices, dtype=np.int64).reshape(-1)
    if idx.size and (idx.min() < 0 or idx.max() >= rows):
        raise BoundsError(f"row index out of range for table {table_id} ({rows} rows)")
    return idx


class DirtyBitmap:
    """One table's bitset in HBM (tracker.py:19-70)."""

    def __init__(self, table_id: int, rows: int, device=None, *, _words: torch.Tensor | None = None,
                 _flags: torch.Tensor | None = None):
        self.table_id = table_id
        self.rows = rows
        dev = device_of(device if _words is None else _words.device)
        self._words = (_words if _words is not None
                       else torch.zeros(_words_for(rows), dtype=torch.int32, device=dev))
        self._flags = _flags if _flags is not None else new_flags(dev)

    @property
    def device(self) -> torch.device:
        return self._words.device

    @property
    def words(self) -> torch.Tensor:
        """The uint32 words (stored as int32) backing the bitmap."""
        return self._words

    def mark(self, indices) -> None:
        """Set the bits of the given rows; repeats are idempotent (tracker.py:27-36)."""
        L = _lib.lib()
        if isinstance(indices, torch.Tensor) and indices.is_cuda:
            idx = indices.to(self.device).to(torch.int64).contiguous().reshape(-1)
        else:
            host = _host_ids(indices, self.rows, self.table_id)
            if host.size == 0:
                return
            idx = torch.from_numpy(host).to(self.device)
        if idx.numel() == 0:
            return
        _lib.check(L.ds_mark_table(self._words.data_ptr(), self.rows, idx.data_ptr(), idx.numel(),
                                   self._flags.data_ptr(), _lib.stream_handle()), "mark")

    def check(self) -> None:
        """Raise a deferred BoundsError from device-tensor marks."""
        v = int(self._flags.item())
        if v:
            self._flags.zero_()
            _lib.raise_flags(v, f"mark (table {self.table_id})")

    def _same_shape(self, other: "DirtyBitmap") -> None:
        if other.table_id != self.table_id or other.rows != self.rows:
            raise ShapeError("bitmaps cover different tables or lengths")

    def merge_or(self, other: "DirtyBitmap") -> "DirtyBitmap":
        """OR into a new bitmap; inputs untouched (tracker.py:38-44)."""
        self._same_shape(other)
        out = DirtyBitmap(self.table_id, self.rows, self.device)
        _lib.check(_lib.lib().ds_bitmap_op(out._words.data_ptr(), self._words.data_ptr(),
                                           other._words.data_ptr(), self._words.numel(), 0,
                                           _lib.stream_handle()), "merge_or")
        return out

    def merge_in(self, other: "DirtyBitmap") -> None:
        """In-place OR (tracker.py:46-49)."""
        self._same_shape(other)
        _lib.check(_lib.lib().ds_bitmap_op(self._words.data_ptr(), other._words.data_ptr(), None,
                                           self._words.numel(), 1, _lib.stream_handle()),
                   "merge_in")

    def popcount(self) -> int:
        self.check()
        out = torch.zeros(1, dtype=torch.int64, device=self.device)
        _lib.check(_lib.lib().ds_popcount(self._words.data_ptr(), self._words.numel(),
                                          out.data_ptr(), _lib.stream_handle()), "popcount")
        return int(out.item())

    def dirty_rows_device(self) -> torch.Tensor:
        """Ascending int64 dirty ids as a device tensor (K2, one table)."""
        self.check()
        return _capture_words(self._words, None, [self.rows], want_int=True, want_union=False,
                              fold=0)[0][0]

    def dirty_rows(self) -> tuple[np.ndarray, float]:
        """Sorted dirty ids (host int64) and the dirty fraction (tracker.py:54-58)."""
        ids = self.dirty_rows_device().cpu().numpy()
        return ids, ids.size / self.rows

    def clear(self) -> None:
        self._words.zero_()

    def copy(self) -> "DirtyBitmap":
        out = DirtyBitmap(self.table_id, self.rows, self.device)
        out._words.copy_(self._words)
        return out

    def to_bytes(self) -> np.ndarray:
        """The reference's uint8 bitset (same bytes as DirtyBitmap._words)."""
        w = self._words.cpu().numpy().view(np.uint8)
        return w[: (self.rows + 7) // 8].copy()

    @property
    def nbytes(self) -> int:
        """Logical bitset size, (rows+7)//8 bytes (tracker.py:68-70)."""
        return (self.rows + 7) // 8


def _capture_words(interval: torch.Tensor, baseline: torch.Tensor | None, rows: list[int],
                   want_int: bool, want_union: bool, fold: int, word_off: list[int] | None = None):
    """Run ds_capture over a table set laid out in `interval`/`baseline`.

    Returns ([int ids per table], [union ids per table], counts tensor).
    Chunks of at most 64 tables per call.
    """
    L = _lib.lib()
    dev = interval.device
    nt = len(rows)
    if word_off is None:
        word_off = [0]
        for r in rows:
            word_off.append(word_off[-1] + _words_for(r))
    out_int, out_uni = [], []
    stream = _lib.stream_handle()
    for c0 in range(0, nt, _lib.MAX_TABLES):
        c1 = min(nt, c0 + _lib.MAX_TABLES)
        sub_rows = rows[c0:c1]
        base = word_off[c0]
        wo = np.array([w - base for w in word_off[c0:c1 + 1]], dtype=np.int64)
        rw = np.array(sub_rows, dtype=np.int64)
        k = c1 - c0
        counts = torch.zeros(2 * k + 2, dtype=torch.int64, device=dev)
        ws_bytes = int(L.ds_capture_workspace_size(int(wo[-1]), k))
        ws = torch.zeros(ws_bytes, dtype=torch.uint8, device=dev)  # zero before first use
        iv = interval[base:]
        bv = baseline[base:] if baseline is not None else None
        # pass 1: counts only (bitmaps are small: 1/256 of the fp32 rows they
        # cover), so the id buffers are sized exactly
        _lib.check(L.ds_capture(iv.data_ptr(), None if bv is None else bv.data_ptr(),
                                wo.ctypes.data_as(ctypes.c_void_p),
                                rw.ctypes.data_as(ctypes.c_void_p), k, None, None,
                                counts.data_ptr(), 0, ws.data_ptr(), ws_bytes, stream), "capture")
        cnt0 = counts.cpu().numpy()
        ids_i = torch.empty(int(cnt0[k]) if want_int else 0, dtype=torch.int64, device=dev)
        ids_u = torch.empty(int(cnt0[2 * k + 1]) if want_union else 0, dtype=torch.int64,
                            device=dev)
        _lib.check(L.ds_capture(iv.data_ptr(), None if bv is None else bv.data_ptr(),
                                wo.ctypes.data_as(ctypes.c_void_p),
                                rw.ctypes.data_as(ctypes.c_void_p), c1 - c0,
                                ids_i.data_ptr() if want_int else None,
                                ids_u.data_ptr() if want_union else None, counts.data_ptr(), fold,
                                ws.data_ptr(), ws_bytes, stream), "capture")
        cnt = cnt0  # the bitmaps did not change between the passes
        ci, cu = cnt[:k], cnt[k + 1:2 * k + 1]
        oi = np.concatenate([[0], np.cumsum(ci)])
        ou = np.concatenate([[0], np.cumsum(cu)])
        for t in range(k):
            if want_int:
                out_int.append(ids_i[oi[t]:oi[t + 1]])
            if want_union:
                out_uni.append(ids_u[ou[t]:ou[t + 1]])
    return out_int, out_uni


@dataclass(frozen=True)
class TrackerView:
    """Per-table row sets captured in the stall window (tracker.py:73-80)."""

    interval_rows: dict
    baseline_rows: dict
    interval_fraction: float
    baseline_fraction: float


class ModelTracker:
    """Both tracking scopes for every table, in two HBM word buffers (tracker.py:83-139)."""

    def __init__(self, table_rows: dict, device=None):
        dev = device_of(device)
        self._tids = sorted(table_rows)
        self._rows = {tid: int(table_rows[tid]) for tid in self._tids}
        # every table's words start 16-byte aligned (4-word padding, always
        # zero) so K2 moves them with 16-byte loads and stores
        self._word_off = [0]
        for tid in self._tids:
            self._word_off.append(self._word_off[-1] + (_words_for(self._rows[tid]) + 3) // 4 * 4)
        total = self._word_off[-1]
        self._ibuf = torch.zeros(total, dtype=torch.int32, device=dev)
        self._bbuf = torch.zeros(total, dtype=torch.int32, device=dev)
        self._flags = new_flags(dev)
        self._interval = {}
        self._baseline = {}
        for k, tid in enumerate(self._tids):
            w0 = self._word_off[k]
            w1 = w0 + _words_for(self._rows[tid])
            self._interval[tid] = DirtyBitmap(tid, self._rows[tid], _words=self._ibuf[w0:w1],
                                              _flags=self._flags)
            self._baseline[tid] = DirtyBitmap(tid, self._rows[tid], _words=self._bbuf[w0:w1],
                                              _flags=self._flags)
        self._total_rows = sum(self._rows.values())

    @property
    def device(self) -> torch.device:
        return self._ibuf.device

    @property
    def table_ids(self) -> list:
        return list(self._tids)

    def mark(self, table_id: int, indices) -> None:
        self._interval[table_id].mark(indices)

    def mark_batch(self, idx: torch.Tensor, seg_off: np.ndarray, seg_tables: np.ndarray) -> None:
        """K1 over a whole batch: idx[seg_off[s]:seg_off[s+1]] belongs to table
        seg_tables[s] (device int64 ids; one launch per 64 segments).  This is
        the call a fused embedding lookup makes once per step."""
        L = _lib.lib()
        pos = {tid: k for k, tid in enumerate(self._tids)}
        wo = np.array(self._word_off, dtype=np.int64)
        rows = np.array([self._rows[t] for t in self._tids], dtype=np.int64)
        seg_off = np.asarray(seg_off, dtype=np.int64)
        tabs = np.array([pos[int(t)] for t in seg_tables], dtype=np.int32)
        stream = _lib.stream_handle()
        for s0 in range(0, len(tabs), _lib.MAX_TABLES):
            s1 = min(len(tabs), s0 + _lib.MAX_TABLES)
            # table indices are into the full set: pass the full word_off/rows
            # when the set is small, else remap per chunk
            sub_t = tabs[s0:s1]
            uniq = sorted(set(sub_t.tolist()))
            remap = {t: k for k, t in enumerate(uniq)}
            wo_c = np.array([wo[t] for t in uniq], dtype=np.int64)
            rows_c = np.array([rows[t] for t in uniq], dtype=np.int64)
            tab_c = np.array([remap[t] for t in sub_t], dtype=np.int32)
            so = np.ascontiguousarray(seg_off[s0:s1 + 1])
            fn = L.ds_mark_i32 if idx.dtype == torch.int32 else L.ds_mark
            _lib.check(fn(self._ibuf.data_ptr(), wo_c.ctypes.data_as(ctypes.c_void_p),
                                 rows_c.ctypes.data_as(ctypes.c_void_p), idx.data_ptr(),
                                 so.ctypes.data_as(ctypes.c_void_p),
                                 tab_c.ctypes.data_as(ctypes.c_void_p), s1 - s0,
                                 self._flags.data_ptr(), stream), "mark_batch")

    def mark_packed(self, stream: "LookupStream") -> None:
        """K1 over a packed mixed-width lookup stream already on this device
        (LookupStream.to); one launch per 64 segments."""
        L = _lib.lib()
        if stream.buf.device != self.device:
            raise ValueError("mark_packed: move the stream to the tracker's device first")
        pos = {tid: k for k, tid in enumerate(self._tids)}
        tabs = np.array([pos[int(t)] for t in stream.seg_tables], dtype=np.int32)
        for s0 in range(0, len(tabs), _lib.MAX_TABLES):
            s1 = min(len(tabs), s0 + _lib.MAX_TABLES)
            uniq = sorted(set(tabs[s0:s1].tolist()))
            remap = {t: k for k, t in enumerate(uniq)}
            wo_c = np.array([self._word_off[t] for t in uniq], dtype=np.int64)
            rows_c = np.array([self._rows[self._tids[t]] for t in uniq], dtype=np.int64)
            tab_c = np.array([remap[t] for t in tabs[s0:s1]], dtype=np.int32)
            boff = np.ascontiguousarray(stream.seg_byte_off[s0:s1], dtype=np.int64)
            cnt = np.ascontiguousarray(stream.seg_count[s0:s1], dtype=np.int64)
            wid = np.ascontiguousarray(stream.seg_width[s0:s1], dtype=np.int32)
            vp = ctypes.c_void_p
            _lib.check(L.ds_mark_packed(
                self._ibuf.data_ptr(), wo_c.ctypes.data_as(vp), rows_c.ctypes.data_as(vp),
                stream.buf.data_ptr(), boff.ctypes.data_as(vp), cnt.ctypes.data_as(vp),
                wid.ctypes.data_as(vp), tab_c.ctypes.data_as(vp), s1 - s0,
                self._flags.data_ptr(), _lib.stream_handle()), "mark_packed")

    def capture_into(self, ids: torch.Tensor, counts: torch.Tensor | None = None, fold: int = 1,
                     scope: str = "interval") -> torch.Tensor:
        """K2 without any host synchronisation (the stall-window form).

        Writes the chosen scope's local row ids of every table, concatenated in
        table order, into `ids` (capacity >= total rows) and the per-table
        counts into counts[:ntables] (counts[ntables] = total), then folds
        (1: reset_interval, 2: reset_baseline, 0: none).  At most 64 tables.
        With counts=None the capture's own device counts are returned (no
        copy; valid until the next capture_into).
        """
        if len(self._tids) > _lib.MAX_TABLES:
            raise ValueError("capture_into supports at most 64 tables")
        L = _lib.lib()
        nt = len(self._tids)
        if not hasattr(self, "_cap_ws"):
            wo = np.array(self._word_off, dtype=np.int64)
            rows = np.array([self._rows[t] for t in self._tids], dtype=np.int64)
            ws_bytes = int(L.ds_capture_workspace_size(int(wo[-1]), nt))
            self._cap_ws = (wo, rows, torch.zeros(ws_bytes, dtype=torch.uint8, device=self.device))
            self._cap_counts = torch.zeros(2 * nt + 2, dtype=torch.int64, device=self.device)
        wo, rows, ws = self._cap_ws
        union = scope != "interval"
        cnt = self._cap_counts
        _lib.check(L.ds_capture(self._ibuf.data_ptr(), self._bbuf.data_ptr(),
                                wo.ctypes.data_as(ctypes.c_void_p),
                                rows.ctypes.data_as(ctypes.c_void_p), nt,
                                None if union else ids.data_ptr(),
                                ids.data_ptr() if union else None, cnt.data_ptr(), fold,
                                ws.data_ptr(), ws.numel(), _lib.stream_handle()), "capture_into")
        src = cnt[nt + 1:2 * nt + 2] if union else cnt[:nt + 1]
        if counts is None:
            return src  # the capture's own counts (valid until the next capture)
        counts[:nt + 1].copy_(src, non_blocking=True)
        return counts

    def interval_bitmap(self, table_id: int) -> DirtyBitmap:
        return self._interval[table_id]

    def baseline_bitmap(self, table_id: int) -> DirtyBitmap:
        """The stored baseline accumulator (without the live interval)."""
        return self._baseline[table_id]

    def since_baseline(self, table_id: int) -> DirtyBitmap:
        return self._baseline[table_id].merge_or(self._interval[table_id])

    def check(self) -> None:
        v = int(self._flags.item())
        if v:
            self._flags.zero_()
            _lib.raise_flags(v, "mark")

    def capture_device(self, want_interval: bool = True, want_union: bool = True, fold: int = 0):
        """K2 over every table in one pass; device id tensors per table.

        fold=1 also performs reset_interval, fold=2 reset_baseline, in the same
        pass (the engine always follows capture with one of them,
        engine.py:278-280).
        """
        self.check()
        rows = [self._rows[t] for t in self._tids]
        ids_i, ids_u = _capture_words(self._ibuf, self._bbuf, rows, want_interval, want_union,
                                      fold, self._word_off)
        iv = {tid: ids_i[k] for k, tid in enumerate(self._tids)} if want_interval else {}
        uv = {tid: ids_u[k] for k, tid in enumerate(self._tids)} if want_union else {}
        return iv, uv

    def capture(self) -> TrackerView:
        """Both scopes as sorted host id arrays (tracker.py:100-118)."""
        iv, uv = self.capture_device()
        interval = {tid: iv[tid].cpu().numpy() for tid in self._tids}
        baseline = {tid: uv[tid].cpu().numpy() for tid in self._tids}
        n_int = sum(a.size for a in interval.values())
        n_base = sum(a.size for a in baseline.values())
        return TrackerView(interval_rows=interval, baseline_rows=baseline,
                           interval_fraction=n_int / self._total_rows,
                           baseline_fraction=n_base / self._total_rows)

    def reset_interval(self) -> None:
        """Fold interval into baseline, clear interval (tracker.py:120-124)."""
        _lib.check(_lib.lib().ds_bitmap_op(None, self._ibuf.data_ptr(), self._bbuf.data_ptr(),
                                           self._ibuf.numel(), 2, _lib.stream_handle()),
                   "reset_interval")

    def reset_baseline(self) -> None:
        """Both scopes empty (tracker.py:126-130)."""
        _lib.check(_lib.lib().ds_bitmap_op(None, self._ibuf.data_ptr(), self._bbuf.data_ptr(),
                                           self._ibuf.numel(), 3, _lib.stream_handle()),
                   "reset_baseline")

    def mark_baseline(self, table_id: int, indices) -> None:
        """Rebuild the since-baseline scope at restore (tracker.py:132-134)."""
        self._baseline[table_id].mark(indices)

    def nbytes(self) -> int:
        return sum(b.nbytes for b in self._interval.values()) + sum(
            b.nbytes for b in self._baseline.values())


# ---------------------------------------------------------------------------
# packed lookup streams (ds_mark_packed)
# ---------------------------------------------------------------------------

def lookup_width(rows: int) -> int:
    """Bits per id for a table of `rows` rows: ceil(log2(rows)) rounded up to
    a multiple of 4 (a lane's 8 ids then fill whole 32-bit words) and at
    least 4, bit-packed; 32 / 64 for signed int32 / int64 above 2^28 rows."""
    b = (max(1, int(rows - 1).bit_length()) + 3) // 4 * 4
    if b <= 28:
        return b
    return 32 if rows <= 1 << 31 else 64


def pack_ids(a, bits: int) -> np.ndarray:
    """Little-endian (LSB-first) bitstream of ids at `bits` bits each; 32 and
    64 bits are plain int32 / int64 arrays."""
    a = np.asarray(a)
    if bits == 64:
        return np.ascontiguousarray(a, dtype=np.int64).view(np.uint8)
    if bits == 32:
        return np.ascontiguousarray(a, dtype=np.int32).view(np.uint8)
    if bits == 8:
        return np.ascontiguousarray(a, dtype=np.uint8)
    if bits == 16:
        return np.ascontiguousarray(a, dtype=np.uint16).view(np.uint8)
    out = np.zeros((a.size * bits + 7) // 8, dtype=np.uint8)
    shifts = np.arange(bits, dtype=np.uint64)
    blk = 1 << 20  # ids per block (a multiple of 8: every block starts on a byte)
    for i in range(0, a.size, blk):
        v = a[i:i + blk].astype(np.uint64)
        bitsm = ((v[:, None] >> shifts) & np.uint64(1)).astype(np.uint8)
        packed = np.packbits(bitsm.reshape(-1), bitorder="little")
        o = i * bits // 8
        out[o:o + packed.size] = packed
    return out


class LookupStream:
    """One interval's (or batch's) lookups of several tables, each table's
    ids bit-packed at ceil(log2(rows)) bits rounded up to a multiple of 4
    (lookup_width) into one byte buffer with 16-byte-aligned segments.

    This is the wire format of K1's input: a data loader fills it on the host
    (pinned), one H2D copy moves it, and ModelTracker.mark_packed consumes it.
    Segment s = seg_count[s] ids of seg_width[s] bits at seg_byte_off[s],
    all of table seg_tables[s].
    """

    def __init__(self, buf: torch.Tensor, seg_byte_off, seg_count, seg_width, seg_tables):
        self.buf = buf
        self.seg_byte_off = np.asarray(seg_byte_off, dtype=np.int64)
        self.seg_count = np.asarray(seg_count, dtype=np.int64)
        self.seg_width = np.asarray(seg_width, dtype=np.int32)
        self.seg_tables = np.asarray(seg_tables, dtype=np.int64)

    @property
    def nbytes(self) -> int:
        """Bytes of the stream (what one H2D copy moves)."""
        return int(self.buf.numel())

    @staticmethod
    def layout(table_rows: dict, counts: dict):
        """(byte offsets, counts, widths, table ids, total bytes) for {tid: count}."""
        tids = list(counts)
        boff, cnt, wid = [], [], []
        off = 0
        for t in tids:
            w = lookup_width(int(table_rows[t]))
            boff.append(off)
            cnt.append(int(counts[t]))
            wid.append(w)
            off += ((int(counts[t]) * w + 7) // 8 + 15) // 16 * 16
        return boff, cnt, wid, tids, off

    @classmethod
    def pack(cls, lookups: dict, table_rows: dict, pin: bool = True) -> "LookupStream":
        """Host-side packing of {table_id: integer ids} (ids are cast to the
        table's width; out-of-range ids must already have been rejected by
        the caller for widths 1 and 2, where they would wrap)."""
        boff, cnt, wid, tids, total = cls.layout(table_rows, {t: len(v) for t, v in lookups.items()})
        buf = torch.empty(max(16, total), dtype=torch.uint8, pin_memory=pin)
        host = buf.numpy()
        for t, o, n, w in zip(tids, boff, cnt, wid):
            a = np.asarray(lookups[t])
            if w < 32 and a.size and (a.min() < 0 or a.max() >= table_rows[t]):
                raise BoundsError(f"table {t}: row index out of range for a {w}-bit stream")
            p = pack_ids(a, w)
            host[o:o + p.size] = p
        return cls(buf, boff, cnt, wid, tids)

    def to(self, device, out: torch.Tensor | None = None, non_blocking: bool = True) -> "LookupStream":
        """The same stream in device memory (one copy; `out` reuses a buffer)."""
        if out is None:
            out = torch.empty(self.buf.numel(), dtype=torch.uint8, device=device)
        out[:self.buf.numel()].copy_(self.buf, non_blocking=non_blocking)
        return LookupStream(out[:self.buf.numel()], self.seg_byte_off, self.seg_count,
                            self.seg_width, self.seg_tables)
