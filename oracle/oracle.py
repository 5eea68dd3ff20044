"""ctypes front end of the CPU oracle (oracle/deltasnap_oracle.c).

TEST INFRASTRUCTURE ONLY: the checker for the CUDA path.  Only tests/,
__graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
import this module.  The product package (paper_2010_08679_b200) never does.

Each wrapper mirrors one reference function of `deltasnap`
(/root/reference/pkg/src/deltasnap) with the same argument meaning:

    quantize_rows / dequantize_rows / reconstruction_errors   quant.py:93-138
    adaptive_params_rows                                       quant.py:160-209
    pack_code_rows / unpack_code_rows / packed_size            quant.py:372-395
    dirty_rows / mark                                          tracker.py:27-58
    build_section / build_shard_payload                        engine.py:118-189
    apply_section (restore scatter)                            engine.py:459-485
"""

from __future__ import annotations

import ctypes
import math
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libdeltasnap_oracle.so")

HEADER_SIZE = 24
STATUS_NAMES = {1: "ConfigError", 2: "DataError", 3: "ShapeError", 4: "BoundsError",
                5: "FormatError", 6: "IntegrityError"}


class OracleError(Exception):
    def __init__(self, status: int, what: str):
        super().__init__(f"{what}: {STATUS_NAMES.get(status, status)}")
        self.status = status
        self.kind = STATUS_NAMES.get(status, str(status))


def build() -> str:
    """Compile the oracle with its committed Makefile (gcc, no FMA contraction)."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)
    return LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = ctypes.CDLL(LIB_PATH)
        P = ctypes.c_void_p
        I64 = ctypes.c_int64
        I = ctypes.c_int
        D = ctypes.c_double
        sig = {
            "dso_mark": (I, [P, I64, P, I64]),
            "dso_popcount": (I64, [P, I64]),
            "dso_dirty_rows": (I64, [P, I64, P]),
            "dso_or": (None, [P, P, P, I64]),
            "dso_pairwise_sum": (D, [P, I64]),
            "dso_row_minmax": (None, [P, I64, I64, P, P]),
            "dso_quantize_rows": (None, [P, I64, I64, P, P, I, P]),
            "dso_dequantize_rows": (I, [P, I64, I64, P, P, I, P]),
            "dso_reconstruction_errors": (None, [P, I64, I64, P, P, I, P]),
            "dso_adaptive_steps": (I, [I, D]),
            "dso_adaptive_params_rows": (I, [P, I64, I64, I, I, I, P, P, I]),
            "dso_packed_size": (I64, [I64, I]),
            "dso_pack_code_rows": (I, [P, I64, I64, I, P]),
            "dso_unpack_code_rows": (I, [P, I64, I64, I, P]),
            "dso_record_size": (I64, [I64, I, I, I]),
            "dso_build_section": (I, [ctypes.c_uint32, P, I64, I64, P, P, I64, I, I, I, I64,
                                      P, P, I]),
            "dso_apply_section": (I, [P, I64, I, P, I64, I64, P, P]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def _check(status: int, what: str):
    if status:
        raise OracleError(status, what)


def _f32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


# --- tracker ---------------------------------------------------------------

def mark(bits: np.ndarray, rows: int, idx) -> None:
    idx = np.ascontiguousarray(idx, dtype=np.int64)
    _check(lib().dso_mark(_p(bits), rows, _p(idx), idx.size), "mark")


def dirty_rows(bits: np.ndarray, rows: int) -> np.ndarray:
    out = np.empty(rows, dtype=np.int64)
    n = lib().dso_dirty_rows(_p(bits), rows, _p(out))
    return out[:n].copy()


def popcount(bits: np.ndarray) -> int:
    return int(lib().dso_popcount(_p(bits), bits.size))


# --- codec -----------------------------------------------------------------

def pairwise_sum(a) -> float:
    a = np.ascontiguousarray(a, dtype=np.float64)
    return float(lib().dso_pairwise_sum(_p(a), a.size))


def row_minmax(x):
    x = _f32(x)
    n, d = x.shape
    lo = np.empty(n, np.float32)
    hi = np.empty(n, np.float32)
    lib().dso_row_minmax(_p(x), n, d, _p(lo), _p(hi))
    return lo, hi


def quantize_rows(x, mins, maxs, bitwidth: int) -> np.ndarray:
    x = _f32(x)
    n, d = x.shape
    out = np.empty((n, d), np.uint8)
    lib().dso_quantize_rows(_p(x), n, d, _p(_f32(mins)), _p(_f32(maxs)), bitwidth, _p(out))
    return out


def dequantize_rows(codes, mins, maxs, bitwidth: int) -> np.ndarray:
    codes = np.ascontiguousarray(codes, dtype=np.uint8)
    n, d = codes.shape
    out = np.empty((n, d), np.float32)
    _check(lib().dso_dequantize_rows(_p(codes), n, d, _p(_f32(mins)), _p(_f32(maxs)),
                                     bitwidth, _p(out)), "dequantize_rows")
    return out


def reconstruction_errors(x, mins, maxs, bitwidth: int) -> np.ndarray:
    x = _f32(x)
    n, d = x.shape
    out = np.empty(n, np.float64)
    lib().dso_reconstruction_errors(_p(x), n, d, _p(_f32(mins)), _p(_f32(maxs)), bitwidth,
                                    _p(out))
    return out


def adaptive_steps(num_bins: int, ratio: float) -> int:
    return int(lib().dso_adaptive_steps(num_bins, ratio))


def adaptive_params_rows(x, bitwidth: int, num_bins: int, ratio: float, nthreads: int = 1):
    x = _f32(x)
    n, d = x.shape
    lo = np.empty(n, np.float32)
    hi = np.empty(n, np.float32)
    steps = adaptive_steps(num_bins, ratio)
    _check(lib().dso_adaptive_params_rows(_p(x), n, d, bitwidth, num_bins, steps, _p(lo), _p(hi),
                                          nthreads), "adaptive_params_rows")
    return lo, hi


def packed_size(dim: int, bitwidth: int) -> int:
    return (dim * bitwidth + 7) // 8


def pack_code_rows(codes, bitwidth: int) -> np.ndarray:
    codes = np.ascontiguousarray(codes, dtype=np.uint8)
    n, d = codes.shape
    out = np.empty((n, packed_size(d, bitwidth)), np.uint8)
    _check(lib().dso_pack_code_rows(_p(codes), n, d, bitwidth, _p(out)), "pack_code_rows")
    return out


def unpack_code_rows(packed, bitwidth: int, dim: int) -> np.ndarray:
    packed = np.ascontiguousarray(packed, dtype=np.uint8)
    n = packed.shape[0]
    if packed.shape[1] != packed_size(dim, bitwidth):
        raise OracleError(5, "unpack_code_rows size")
    out = np.empty((n, dim), np.uint8)
    _check(lib().dso_unpack_code_rows(_p(packed), n, dim, bitwidth, _p(out)), "unpack_code_rows")
    return out


def record_size(dim: int, bitwidth: int | None, aux: bool, incremental: bool) -> int:
    return int(lib().dso_record_size(dim, bitwidth or 0, int(aux), int(incremental)))


# --- writer / restore --------------------------------------------------------

def build_section(table_id: int, values, sel=None, *, bitwidth: int | None,
                  adaptive: tuple[int, float] | None = None, aux=None, chunk_rows: int = 1024,
                  nthreads: int = 1, err_in: float = 0.0):
    """One table's section bytes (engine.py:139-187 + payload.py:84-104).

    Returns (bytes, q_rows, err_sum) with err_sum = err_in plus the chunk
    errors accumulated in the reference's order for the given chunk_rows.
    """
    values = _f32(values)
    rows, d = values.shape
    aux_a = None if aux is None else _f32(aux)
    sel_a = None if sel is None else np.ascontiguousarray(sel, dtype=np.int64)
    n = rows if sel_a is None else sel_a.size
    bits = bitwidth or 0
    bins, steps = 0, 0
    if bits and adaptive is not None:
        bins = int(adaptive[0])
        steps = adaptive_steps(adaptive[0], adaptive[1])
    rec = record_size(d, bitwidth, aux_a is not None, sel_a is not None)
    out = np.empty(HEADER_SIZE + n * rec, np.uint8)
    err = np.full(1, err_in, np.float64)
    _check(lib().dso_build_section(table_id, _p(values), rows, d, _p(aux_a), _p(sel_a), n, bits,
                                   bins, steps, chunk_rows, _p(out), _p(err), nthreads),
           "build_section")
    return out.tobytes(), (n if bits else 0), float(err[0])


def build_shard_payload(tables: dict, plan_kind: str, plan_rows, bitwidth, shard_tables,
                        chunk_rows: int = 1024, adaptive=None, nthreads: int = 1):
    """build_shard_payload (engine.py:118-189) over an explicit table list.

    tables: {tid: (values, aux|None)}; shard_tables: sorted tids of the shard;
    adaptive: {bitwidth: (bins, ratio)} overrides merged over DEFAULT_ADAPTIVE.
    """
    defaults = {2: (25, 0.5), 3: (25, 0.2), 4: (45, 0.2)}
    if adaptive:
        defaults.update(adaptive)
    acfg = defaults.get(bitwidth) if bitwidth is not None else None
    parts, q_rows, err_sum = [], 0, 0.0
    for tid in shard_tables:
        values, aux = tables[tid]
        sel = None
        if plan_kind == "incremental":
            sel = plan_rows.get(tid)
            sel = np.zeros(0, np.int64) if sel is None else sel
        blob, q, err_sum = build_section(tid, values, sel, bitwidth=bitwidth, adaptive=acfg,
                                         aux=aux, chunk_rows=chunk_rows, nthreads=nthreads,
                                         err_in=err_sum)
        parts.append(blob)
        q_rows += q
    return b"".join(parts), q_rows, err_sum


def apply_section(section: bytes, incremental: bool, values: np.ndarray, aux=None,
                  baseline_bits=None) -> None:
    buf = np.frombuffer(section, dtype=np.uint8)
    rows, d = values.shape
    _check(lib().dso_apply_section(_p(buf), buf.size, int(incremental), _p(values), rows, d,
                                   _p(aux), _p(baseline_bits)), "apply_section")


def split_sections(payload: bytes, incremental: bool):
    """Walk a shard payload into (table_id, section_bytes) pieces (payload.py:111-164)."""
    import struct
    out = []
    off = 0
    while off < len(payload):
        if len(payload) - off < HEADER_SIZE:
            raise OracleError(5, "truncated section header")
        magic, tid, rows, dim, bw, mode, auxf, rsv = struct.unpack_from("<4sIQIBBBB", payload, off)
        if magic != b"CNR1" or mode not in (0, 1) or rsv != 0 or auxf not in (0, 1) or dim < 1:
            raise OracleError(5, "bad header")
        rec = record_size(dim, bw if mode == 1 else None, bool(auxf), incremental)
        end = off + HEADER_SIZE + rows * rec
        if end > len(payload):
            raise OracleError(5, "truncated section body")
        out.append((tid, payload[off:end]))
        off = end
    return out


def nan_safe_equal_params(a: np.ndarray, b: np.ndarray) -> bool:
    """Equality with +0 == -0 (the documented signed-zero exception)."""
    return bool(np.array_equal(np.asarray(a, np.float32), np.asarray(b, np.float32)))


def default_steps(bitwidth: int) -> int:
    table = {2: (25, 0.5), 3: (25, 0.2), 4: (45, 0.2)}
    b, r = table[bitwidth]
    return int(math.floor(b * r + 1e-9))
