"""ctypes binding of libdeltasnap_cuda.so (include/deltasnap_cuda.h).

The product path has exactly one backend: the sm_100a kernels in this
library.  If the library or a CUDA device is missing, every entry point
raises -- there is no CPU fallback.
"""

from __future__ import annotations

import ctypes
import os
import threading

import torch

from . import errors

HERE = os.path.dirname(os.path.abspath(__file__))
# DS_CUDA_LIB selects an A/B build variant of the same library (csrc/Makefile)
LIB_PATH = os.environ.get("DS_CUDA_LIB") or os.path.join(HERE, "libdeltasnap_cuda.so")

# ds_status -> exception (include/deltasnap_cuda.h; deltasnap/errors.py:4-41)
_STATUS = {
    1: errors.ConfigError,
    2: errors.DataError,
    3: errors.ShapeError,
    4: errors.BoundsError,
    5: errors.FormatError,
    6: errors.IntegrityError,
}
FLAG_BOUNDS = 0x1
FLAG_DATA = 0x2
FLAG_FORMAT = 0x4
FLAG_INTEGRITY = 0x8
FLAG_CAPACITY = 0x10
FLAG_TIMEOUT = 0x20

STAT_EXACT_DECISIONS = 0
STAT_EXACT_CODES = 1
STAT_ROWS = 2
STAT_COUNT = 4

MAX_TABLES = 64


class TableDesc(ctypes.Structure):
    _fields_ = [
        ("values", ctypes.c_void_p),
        ("aux", ctypes.c_void_p),
        ("ld", ctypes.c_int64),
        ("rows", ctypes.c_int64),
        ("row_base", ctypes.c_int64),
        ("ids_off", ctypes.c_int64),
        ("table_id", ctypes.c_uint32),
        ("dim", ctypes.c_uint32),
    ]


class CkptParams(ctypes.Structure):
    _fields_ = [
        ("bitwidth", ctypes.c_int),
        ("incremental", ctypes.c_int),
        ("adaptive_bins", ctypes.c_int),
        ("adaptive_steps", ctypes.c_int),
        ("write_headers", ctypes.c_int),
        ("aux", ctypes.c_int),
        ("ids_packed", ctypes.c_int),
        ("ids_local", ctypes.c_int),
        ("stats", ctypes.c_void_p),
        ("staged", ctypes.c_void_p),
        ("exchange", ctypes.c_void_p),
        ("staged_rows", ctypes.c_int64),
    ]


PEER_MAX = 64


class PeerExchange(ctypes.Structure):
    """ds_peer_exchange: the row-sharded count exchange run inside K3."""
    _fields_ = [
        ("peers", ctypes.c_void_p * PEER_MAX),
        ("out", ctypes.c_void_p),
        ("flags", ctypes.c_void_p),
        ("timeout_ns", ctypes.c_int64),
        ("world", ctypes.c_int),
        ("rank", ctypes.c_int),
        ("epoch", ctypes.c_uint32),
    ]


class TrainTable(ctypes.Structure):
    _fields_ = [
        ("values", ctypes.c_void_p),
        ("aux", ctypes.c_void_p),
        ("words", ctypes.c_void_p),
        ("ld", ctypes.c_int64),
        ("rows", ctypes.c_int64),
    ]


class RestoreSec(ctypes.Structure):
    _fields_ = [
        ("body_off", ctypes.c_int64),
        ("nrec", ctypes.c_int64),
        ("values", ctypes.c_void_p),
        ("aux_values", ctypes.c_void_p),
        ("baseline", ctypes.c_void_p),
        ("ld", ctypes.c_int64),
        ("table_rows", ctypes.c_int64),
        ("row_lo", ctypes.c_int64),
        ("row_hi", ctypes.c_int64),
    ]


_P = ctypes.c_void_p
_I64 = ctypes.c_int64
_I = ctypes.c_int
_SZ = ctypes.c_size_t

_SIGNATURES = {
    "ds_version": (ctypes.c_char_p, []),
    "ds_last_error": (ctypes.c_char_p, []),
    "ds_device_sm_count": (_I, [_I]),
    "ds_set_l2_fetch_granularity": (_I, [_I]),
    "ds_get_l2_fetch_granularity": (_I, []),
    "ds_mark": (_I, [_P, _P, _P, _P, _P, _P, _I, _P, _P]),
    "ds_mark_i32": (_I, [_P, _P, _P, _P, _P, _P, _I, _P, _P]),
    "ds_mark_packed": (_I, [_P, _P, _P, _P, _P, _P, _P, _P, _I, _P, _P]),
    "ds_mark_table": (_I, [_P, _I64, _P, _I64, _P, _P]),
    "ds_bitmap_op": (_I, [_P, _P, _P, _I64, _I, _P]),
    "ds_popcount": (_I, [_P, _I64, _P, _P]),
    "ds_capture_workspace_size": (_SZ, [_I64, _I]),
    "ds_capture": (_I, [_P, _P, _P, _P, _I, _P, _P, _P, _I, _P, _SZ, _P]),
    "ds_writer_workspace_size": (_SZ, [_I, _I64, _I64]),
    "ds_write_payload": (_I, [_P, _I, _P, _P, _P, _P, _I64, _P, _P, _P, _P, _SZ, _P]),
    "ds_record_size": (_I64, [_I64, _I, _I, _I]),
    "ds_stage_rows": (_I, [_P, _I, _P, _P, _I64, _P, _P, _P]),
    "ds_restore_section": (_I, [_P, _I64, _I64, _I, _I, _I, _I64, _I64, _I64, _P, _I64, _P, _P,
                                _P, _P]),
    "ds_restore_payload": (_I, [_P, _P, _I, _I64, _I, _I, _I, _P, _P]),
    "ds_train_apply": (_I, [_P, _I, _I, _I64, _P, _P, _P, _P, _P]),
    "ds_train_apply_sorted": (_I, [_P, _I, _P, _I64, _P, _P, _P, _P, _P]),
    "ds_train_interval_workspace_size": (_SZ, [_I64]),
    "ds_train_interval_delta_bytes": (_SZ, [_I64, _I64]),
    "ds_train_apply_interval": (_I, [_P, _I, _P, _I64, _P, _P, _P, _SZ, _P, _P]),
    "ds_sort_workspace_size": (_SZ, [_I64]),
    "ds_sort_pairs_u32": (_I, [_P, _P, _P, _P, _I64, _I, _P, _SZ, _P]),
    "ds_crc32_workspace_size": (_SZ, [_I64]),
    "ds_crc32": (_I, [_P, _I64, _P, _P, _SZ, _P]),
    "ds_peer_buffer_size": (_SZ, [_I, _I]),
    "ds_peer_alloc": (_I, [_SZ, _P, _P]),
    "ds_peer_open": (_I, [_P, _P]),
    "ds_peer_close": (_I, [_P]),
    "ds_peer_free": (_I, [_P]),
    "ds_quantize_rows": (_I, [_P, _I64, _I64, _P, _P, _I, _P, _P]),
    "ds_dequantize_rows": (_I, [_P, _I64, _I64, _P, _P, _I, _P, _P, _P]),
    "ds_reconstruction_errors": (_I, [_P, _I64, _I64, _P, _P, _I, _P, _P]),
    "ds_adaptive_params_rows": (_I, [_P, _I64, _I64, _I, _I, _I, _P, _P, _P, _P, _P]),
    "ds_row_minmax": (_I, [_P, _I64, _I64, _P, _P, _P]),
    "ds_pack_code_rows": (_I, [_P, _I64, _I64, _I, _P, _P, _P]),
    "ds_unpack_code_rows": (_I, [_P, _I64, _I64, _I, _P, _P, _P]),
}

_lock = threading.Lock()
_lib = None


def lib():
    """Load the CUDA library; raise if it or a CUDA device is unavailable."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
                "g.build()'` (make -C paper_2010_08679_b200/csrc). There is no CPU fallback.")
        L = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in _SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def require_cuda() -> None:
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2010_08679_b200 needs a CUDA device (B200, sm_100a); "
                           "there is no CPU fallback")


def last_error() -> str:
    msg = lib().ds_last_error()
    return msg.decode() if msg else ""


def check(status: int, what: str) -> None:
    if status == 0:
        return
    text = last_error()
    exc = _STATUS.get(status)
    if exc is not None:
        raise exc(f"{what}: {text}")
    if status == 7:
        raise RuntimeError(f"{what}: CUDA error: {text}")
    raise ValueError(f"{what}: invalid argument: {text}")


def raise_flags(flags: int, what: str) -> None:
    """Raise the reference exception for device flag bits (checked at sync).

    Precedence follows the reference's order of checks: a malformed payload
    (FormatError) is detected by decode before the row bounds
    (IntegrityError, engine.py:459-472).
    """
    if not flags:
        return
    if flags & FLAG_TIMEOUT:
        raise RuntimeError(f"{what}: a rank never published its counts (peer exchange timed out)")
    if flags & FLAG_CAPACITY:
        raise ValueError(f"{what}: output buffer too small")
    if flags & FLAG_FORMAT:
        raise errors.FormatError(f"{what}: nonzero padding bits or code out of range")
    if flags & FLAG_DATA:
        raise errors.DataError(f"{what}: vector contains NaN or Inf")
    if flags & FLAG_BOUNDS:
        raise errors.BoundsError(f"{what}: row index out of range")
    if flags & FLAG_INTEGRITY:
        raise errors.IntegrityError(f"{what}: row index out of range")


def ptr(t) -> int | None:
    if t is None:
        return None
    return t.data_ptr()


def stream_handle(stream=None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def version() -> str:
    return lib().ds_version().decode()
