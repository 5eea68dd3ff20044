"""At-scale parity checks of device-written shard payloads against the oracle.

TEST INFRASTRUCTURE (like the rest of oracle/): imported only by tests/,
__graft_entry__.smoke() and bench.py's verification leg, as the checker of
payloads the CUDA path already produced -- never as the thing measured.

Rows are independent through the whole codec (quant.py:14-15 upstream;
SPEC.md:271), so a payload of any size is checked by
  * every section header (payload.py:88-91) against the expected table id,
    record count, dim, bitwidth/mode and aux flag;
  * the FULL dirty-id column of incremental sections against the expected
    sorted dirty set (tracker.py:54-58: np.unique of the interval's lookups);
  * the record bytes (params + packed codes, or fp32 values) of a sample:
    an even stride over all records, the first and last record of every
    section, and every record within a window around the byte offsets
    2^31 and 2^32 (64-bit offset arithmetic), each recomputed by the oracle
    (oracle/deltasnap_oracle.c, build_section) from the same rows.
"""

from __future__ import annotations

import os
import struct
import time

import numpy as np

from . import oracle as O

HEADER_SIZE = 24


def _sections(payload: np.ndarray, incremental: bool):
    """(offset, table_id, rows, dim, bitwidth, mode, aux, rec) per section."""
    out, off, n = [], 0, int(payload.size)
    raw = memoryview(payload)
    while off < n:
        if n - off < HEADER_SIZE:
            raise ValueError(f"truncated header at byte {off}")
        magic, tid, rows, dim, bw, mode, aux, rsv = struct.unpack_from("<4sIQIBBBB", raw, off)
        if magic != b"CNR1" or mode not in (0, 1) or rsv != 0 or aux not in (0, 1) or dim < 1:
            raise ValueError(f"bad header at byte {off}")
        rec = O.record_size(dim, bw if mode == 1 else None, bool(aux), incremental)
        out.append((off, tid, rows, dim, bw, mode, aux, rec))
        off += HEADER_SIZE + rows * rec
        if off > n:
            raise ValueError("truncated section body")
    return out


def verify_payload(payload, expected: list, *, bitwidth: int | None, adaptive=None,
                   incremental: bool, fetch_rows, sample: int = 1_000_000,
                   windows=(1 << 31, 1 << 32), window_records: int = 4096,
                   nthreads: int | None = None) -> dict:
    """Check one shard payload (host uint8 array or bytes).

    expected: per section in payload order, dict(table_id, dim, ids) with
    ids the sorted int64 dirty rows (incremental) or rows=int (full).
    fetch_rows(table_id, ids) -> float32 [len(ids), dim] host rows (the table
    contents the writer read).  adaptive: (num_bins, ratio) or None (naive).
    Returns counts and the number of mismatches (0 = parity).
    """
    t0 = time.perf_counter()
    payload = np.frombuffer(payload, np.uint8) if not isinstance(payload, np.ndarray) else payload
    nthreads = nthreads or os.cpu_count() or 1
    secs = _sections(payload, incremental)
    res = {"headers_checked": 0, "ids_checked": 0, "records_checked": 0,
           "records_past_2^31_checked": 0, "mismatches": 0, "first_mismatch": None,
           "payload_bytes": int(payload.size)}

    def bad(what):
        res["mismatches"] += 1
        if res["first_mismatch"] is None:
            res["first_mismatch"] = what

    if len(secs) != len(expected):
        bad(f"{len(secs)} sections, expected {len(expected)}")
        return res
    mode_want = 1 if bitwidth else 0
    bw_want = bitwidth if bitwidth else 32
    # global record numbering for the sample
    starts, total = [], 0
    for s in secs:
        starts.append(total)
        total += s[2]
    picks = set(range(0, total, max(1, total // max(1, sample))))
    for (off, tid, rows, dim, bw, mode, aux, rec), g0 in zip(secs, starts):
        if rows:
            picks.update((g0, g0 + rows - 1))
        for w in windows:  # records around a byte offset past 2^31 / 2^32
            body0 = off + HEADER_SIZE
            if body0 <= w < body0 + rows * rec:
                k = (w - body0) // rec
                picks.update(range(g0 + max(0, k - window_records // 2),
                                   g0 + min(rows, k + window_records // 2)))
    picks = np.array(sorted(picks), np.int64)

    for k, ((off, tid, rows, dim, bw, mode, aux, rec), exp) in enumerate(zip(secs, expected)):
        res["headers_checked"] += 1
        want_rows = exp["ids"].size if incremental else int(exp["rows"])
        if (tid, rows, dim, bw, mode, aux) != (exp["table_id"], want_rows, exp["dim"], bw_want,
                                               mode_want, int(exp.get("aux", 0))):
            bad(f"header of section {k}: {(tid, rows, dim, bw, mode, aux)}")
            continue
        body = payload[off + HEADER_SIZE: off + HEADER_SIZE + rows * rec].reshape(rows, rec)
        if incremental:
            ids = body[:, :8].copy().view("<u8").reshape(-1).astype(np.int64)
            res["ids_checked"] += int(ids.size)
            nbad = int(np.count_nonzero(ids != exp["ids"]))
            if nbad:
                bad(f"table {tid}: {nbad} dirty ids differ")
        g0 = starts[k]
        sel = picks[(picks >= g0) & (picks < g0 + rows)] - g0
        if sel.size == 0:
            continue
        row_ids = exp["ids"][sel] if incremental else sel
        x = np.ascontiguousarray(fetch_rows(tid, row_ids), dtype=np.float32)
        want, _, _ = O.build_section(tid, x, None, bitwidth=bitwidth, adaptive=adaptive,
                                     nthreads=nthreads)
        want = np.frombuffer(want, np.uint8)[HEADER_SIZE:].reshape(sel.size, rec - (8 if incremental else 0))
        got = body[sel, 8:] if incremental else body[sel]
        diff = np.any(got != want, axis=1)
        if bitwidth and diff.any():
            # the one documented exception: the sign of a zero range endpoint
            # (numpy's SIMD min/max): compare params as floats
            d_idx = np.nonzero(diff)[0]
            gp = got[d_idx, :8].copy().view(np.float32)
            wp = want[d_idx, :8].copy().view(np.float32)
            only_zero = np.all(gp == wp, axis=1) & np.all(got[d_idx, 8:] == want[d_idx, 8:], axis=1)
            diff[d_idx[only_zero]] = False
        res["records_checked"] += int(sel.size)
        past = off + HEADER_SIZE + sel * rec >= (1 << 31)
        res["records_past_2^31_checked"] += int(np.count_nonzero(past))
        if diff.any():
            j = int(np.nonzero(diff)[0][0])
            res["mismatches"] += int(diff.sum()) - 1
            bad(f"table {tid} record {int(sel[j])} (row {int(row_ids[j])}) differs")
    res["seconds"] = time.perf_counter() - t0
    return res
