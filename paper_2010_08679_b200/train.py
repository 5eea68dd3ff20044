"""The synthetic training step with tracking folded in.

Mirror of deltasnap/sim.py:140-155 apply_batch: per table, values[idx] +=
delta, aux[idx] += delta * delta with np.add.at's semantics (bit-identical
float sums for repeated rows) and tracker.mark(tid, idx) -- one launch
(ds_train_apply) for any number of batches, the dirty bits set by the same
thread that updates each distinct row.
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _lib
from ._device import check_flags, new_flags, to_device

MAX_IDS_PER_BATCH = 4096  # ds_train_apply's per-(table, batch) sort capacity (sorted_runs=False)


def pack_batches(tables: dict, batches: list, device=None):
    """Device (idx, delta, seg_off, nbatches) of `batches` (each {table_id:
    (idx, delta)}), table-major then batch order -- ds_train_apply's input."""
    tids = sorted(tables)
    dev = tables[tids[0]].values.device if device is None else torch.device(device)
    dim = tables[tids[0]].dim
    if any(tables[t].dim != dim for t in tids):
        raise ValueError("apply_batches: tables of one call share dim")
    idx_parts, delta_parts, seg = [], [], [0]
    for t in tids:
        for batch in batches:
            ids, dl = batch.get(t, (np.zeros(0, np.int64), np.zeros((0, dim), np.float32)))
            n = len(ids)
            if n > MAX_IDS_PER_BATCH:
                raise ValueError(f"apply_batches: {n} ids for table {t} in one batch "
                                 f"(at most {MAX_IDS_PER_BATCH})")
            idx_parts.append(to_device(ids, torch.int64, dev).reshape(-1))
            delta_parts.append(to_device(dl, torch.float32, dev).reshape(n, dim))
            seg.append(seg[-1] + n)
    idx = torch.cat(idx_parts) if seg[-1] else torch.zeros(1, dtype=torch.int64, device=dev)
    delta = torch.cat(delta_parts) if seg[-1] else torch.zeros((1, dim), device=dev)
    seg_off = torch.tensor(seg, dtype=torch.int64, device=dev)
    return PackedBatches((idx, delta, seg_off, len(batches)), np.asarray(seg, np.int64))


class PackedBatches(tuple):
    """(idx, delta, seg_off, nbatches) with the host copy of seg_off."""

    def __new__(cls, items, host_seg):
        obj = super().__new__(cls, items)
        obj.host_seg = host_seg
        return obj


def apply_packed(tables: dict, packed, tracker=None, sorted_runs: bool = True) -> None:
    """pack_batches' output applied on the device (asynchronous; with a
    tracker, id errors surface at its next sync like mark_batch).

    sorted_runs (default): the whole interval in one pass -- an in-tree
    stable radix sort of (table, row) keys groups each row's updates in array
    order, then a warp per run applies them (ds_train_apply_interval); else
    ds_train_apply (a CTA per table walking the batches with a shared-memory
    sort per batch)."""
    idx, delta, seg_off, nb = packed
    tids = sorted(tables)
    dim = tables[tids[0]].dim
    descs = (_lib.TrainTable * len(tids))()
    for k, t in enumerate(tids):
        tb = tables[t]
        descs[k].values = tb.values.data_ptr()
        descs[k].aux = tb.aux.data_ptr() if tb.aux is not None else None
        descs[k].words = tracker.interval_bitmap(t).words.data_ptr() if tracker is not None else None
        descs[k].ld = tb.values.stride(0)
        descs[k].rows = tb.rows
    flags = tracker._flags if tracker is not None else new_flags(idx.device)
    L = _lib.lib()
    if sorted_runs:
        seg = packed_table_offsets(packed, len(tids))
        n = int(seg[-1])
        nbytes = int(L.ds_train_interval_workspace_size(n)) + int(L.ds_train_interval_delta_bytes(n, dim))
        ws = torch.empty(max(1, nbytes), dtype=torch.uint8, device=idx.device)
        _lib.check(L.ds_train_apply_interval(
            ctypes.cast(descs, ctypes.c_void_p), len(tids), seg.ctypes.data_as(ctypes.c_void_p), dim,
            idx.data_ptr(), delta.data_ptr(), ws.data_ptr(), ws.numel(), flags.data_ptr(),
            _lib.stream_handle()), "train_apply_interval")
    else:
        _lib.check(L.ds_train_apply(ctypes.cast(descs, ctypes.c_void_p), len(tids), nb, dim,
                                    idx.data_ptr(), delta.data_ptr(), seg_off.data_ptr(),
                                    flags.data_ptr(), _lib.stream_handle()), "train_apply")
    if tracker is None:
        check_flags(flags, "apply_batches")


def packed_table_offsets(packed, ntables: int) -> np.ndarray:
    """Host int64 [ntables + 1]: table t's lookups of a packed interval.
    (pack_batches keeps the host copy; a device seg_off is read once.)"""
    idx, delta, seg_off, nb = packed
    seg = getattr(packed, "host_seg", None)
    if seg is None:
        seg = seg_off.cpu().numpy()
    return np.array([seg[k * nb] for k in range(ntables)] + [seg[-1]], dtype=np.int64)


def apply_batches(tables: dict, batches: list, tracker=None, device=None) -> None:
    """Apply `batches` in order (each {table_id: (idx, delta)} like
    sim.generate_batch) to device tables {table_id: DeviceTable}; with a
    ModelTracker the touched rows are marked in its interval scope."""
    if not batches:
        return
    apply_packed(tables, pack_batches(tables, batches, device), tracker)
