"""Per-row uniform codec on the GPU (quant.py API mirror).

Same names, argument meaning, return types and exceptions as
deltasnap/quant.py:26-412 for the checkpoint-path codec; every numeric
function runs in an sm_100a kernel (ds_codec.cu / ds_common.cuh) and returns
results bit-identical to the reference's float64 numpy arithmetic.  Inputs may
be numpy arrays (results come back as numpy, like the reference) or CUDA
tensors (results stay on the device).

Out of scope (benchmark-only in the reference, quant.py:10-12): the k-means
codecs.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._device import check_flags, device_of, like_input, new_flags, to_device
from .errors import ConfigError, DataError, FormatError, ShapeError

VALID_BITWIDTHS = (2, 3, 4, 8)

# greedy search defaults per bitwidth (bins, ratio); 8-bit uses naive ranges
# (quant.py:30)
DEFAULT_ADAPTIVE = {2: (25, 0.5), 3: (25, 0.2), 4: (45, 0.2)}


def _f32(v: float) -> float:
    return float(np.float32(v))


@dataclass(frozen=True)
class QuantParams:
    """Range of one vector, held at float32 precision (quant.py:33-61)."""

    bitwidth: int
    x_min: float
    x_max: float

    def __post_init__(self):
        if self.bitwidth not in VALID_BITWIDTHS:
            raise ConfigError(f"bitwidth must be one of {VALID_BITWIDTHS}")
        if not (math.isfinite(self.x_min) and math.isfinite(self.x_max)):
            raise DataError("quantization range must be finite")
        if self.x_min > self.x_max:
            raise DataError("x_min must not exceed x_max")
        object.__setattr__(self, "x_min", _f32(self.x_min))
        object.__setattr__(self, "x_max", _f32(self.x_max))

    @property
    def scale(self) -> float:
        return (self.x_max - self.x_min) / (2 ** self.bitwidth - 1)

    @property
    def zero_point(self) -> float:
        return self.x_min


@dataclass(frozen=True)
class QuantizedVector:
    params: QuantParams
    codes: np.ndarray


@dataclass(frozen=True)
class AdaptiveConfig:
    """Greedy search knobs (quant.py:141-150)."""

    num_bins: int
    ratio: float

    def __post_init__(self):
        if self.num_bins < 1:
            raise ConfigError("num_bins must be >= 1")
        if not (0 < self.ratio <= 1):
            raise ConfigError("ratio must be in (0, 1]")

    @property
    def steps(self) -> int:
        """floor(num_bins * ratio + 1e-9) greedy steps (quant.py:186)."""
        return int(math.floor(self.num_bins * self.ratio + 1e-9))


def default_adaptive_config(bitwidth: int) -> AdaptiveConfig | None:
    if bitwidth in DEFAULT_ADAPTIVE:
        return AdaptiveConfig(*DEFAULT_ADAPTIVE[bitwidth])
    return None


def _check_bitwidth(bitwidth: int) -> None:
    if bitwidth not in VALID_BITWIDTHS:
        raise ConfigError(f"bitwidth must be one of {VALID_BITWIDTHS}")


def _rows_2d(x, dev, dtype=torch.float32):
    t = to_device(x, dtype, dev)
    if t.dim() != 2:
        raise ShapeError("expected a (rows, dim) matrix")
    return t


def _dev_for(x):
    return device_of(x.device if isinstance(x, torch.Tensor) and x.is_cuda else None)


def row_minmax(x):
    """Naive ranges: x.min(axis=1), x.max(axis=1) (engine.py:163-164)."""
    dev = _dev_for(x)
    t = _rows_2d(x, dev)
    n, d = t.shape
    mins = torch.empty(n, dtype=torch.float32, device=dev)
    maxs = torch.empty(n, dtype=torch.float32, device=dev)
    _lib.check(_lib.lib().ds_row_minmax(t.data_ptr(), n, d, mins.data_ptr(), maxs.data_ptr(),
                                        _lib.stream_handle()), "row_minmax")
    return like_input(mins, x), like_input(maxs, x)


def quantize_rows(x, mins, maxs, bitwidth: int):
    """(rows, dim) uint8 codes; scale-0 rows give all-zero codes (quant.py:93-106)."""
    _check_bitwidth(bitwidth)
    dev = _dev_for(x)
    t = _rows_2d(x, dev)
    n, d = t.shape
    lo = to_device(mins, torch.float32, dev).reshape(-1)
    hi = to_device(maxs, torch.float32, dev).reshape(-1)
    codes = torch.empty((n, d), dtype=torch.uint8, device=dev)
    _lib.check(_lib.lib().ds_quantize_rows(t.data_ptr(), n, d, lo.data_ptr(), hi.data_ptr(),
                                           bitwidth, codes.data_ptr(), _lib.stream_handle()),
               "quantize_rows")
    return like_input(codes, x)


def dequantize_rows(codes, mins, maxs, bitwidth: int):
    """scale * code + zero_point as float32 (quant.py:109-115)."""
    _check_bitwidth(bitwidth)
    dev = _dev_for(codes)
    c = _rows_2d(codes, dev, torch.uint8)
    n, d = c.shape
    lo = to_device(mins, torch.float32, dev).reshape(-1)
    hi = to_device(maxs, torch.float32, dev).reshape(-1)
    out = torch.empty((n, d), dtype=torch.float32, device=dev)
    flags = new_flags(dev)
    _lib.check(_lib.lib().ds_dequantize_rows(c.data_ptr(), n, d, lo.data_ptr(), hi.data_ptr(),
                                             bitwidth, out.data_ptr(), flags.data_ptr(),
                                             _lib.stream_handle()), "dequantize_rows")
    if int(flags.item()):
        raise FormatError(f"code out of range for bitwidth {bitwidth}")
    return like_input(out, codes)


def reconstruction_errors(x, mins, maxs, bitwidth: int):
    """Per-row float64 L2 of x - dequantize(quantize(x)), in numpy's summation
    order (quant.py:134-138)."""
    _check_bitwidth(bitwidth)
    dev = _dev_for(x)
    t = _rows_2d(x, dev)
    n, d = t.shape
    lo = to_device(mins, torch.float32, dev).reshape(-1)
    hi = to_device(maxs, torch.float32, dev).reshape(-1)
    out = torch.empty(n, dtype=torch.float64, device=dev)
    _lib.check(_lib.lib().ds_reconstruction_errors(t.data_ptr(), n, d, lo.data_ptr(),
                                                   hi.data_ptr(), bitwidth, out.data_ptr(),
                                                   _lib.stream_handle()),
               "reconstruction_errors")
    return like_input(out, x)


def adaptive_params_rows(x, bitwidth: int, cfg: AdaptiveConfig, stats: torch.Tensor | None = None):
    """Greedy range search per row (quant.py:160-209); float32 (mins, maxs).

    `stats` (optional int64 device tensor of length >= 4) receives the count
    of decisions that the certified fp32 path re-took in exact float64.
    """
    _check_bitwidth(bitwidth)
    dev = _dev_for(x)
    t = _rows_2d(x, dev)
    n, d = t.shape
    mins = torch.empty(n, dtype=torch.float32, device=dev)
    maxs = torch.empty(n, dtype=torch.float32, device=dev)
    flags = new_flags(dev)
    _lib.check(_lib.lib().ds_adaptive_params_rows(
        t.data_ptr(), n, d, bitwidth, cfg.num_bins, cfg.steps, mins.data_ptr(), maxs.data_ptr(),
        flags.data_ptr(), None if stats is None else stats.data_ptr(), _lib.stream_handle()),
        "adaptive_params_rows")
    if int(flags.item()):
        raise DataError("vector contains NaN or Inf")
    return like_input(mins, x), like_input(maxs, x)


def packed_size(dim: int, bitwidth: int) -> int:
    return (dim * bitwidth + 7) // 8


def pack_code_rows(codes, bitwidth: int):
    """LSB-first bit-packing of a (rows, dim) code matrix (quant.py:376-382)."""
    _check_bitwidth(bitwidth)
    dev = _dev_for(codes)
    c = _rows_2d(codes, dev, torch.uint8)
    n, d = c.shape
    out = torch.empty((n, packed_size(d, bitwidth)), dtype=torch.uint8, device=dev)
    flags = new_flags(dev)
    _lib.check(_lib.lib().ds_pack_code_rows(c.data_ptr(), n, d, bitwidth, out.data_ptr(),
                                            flags.data_ptr(), _lib.stream_handle()),
               "pack_code_rows")
    if int(flags.item()):
        raise DataError(f"code out of range for bitwidth {bitwidth}")
    return like_input(out, codes)


def unpack_code_rows(packed, bitwidth: int, dim: int):
    """Inverse of pack_code_rows; checks width and zero padding (quant.py:385-395)."""
    _check_bitwidth(bitwidth)
    dev = _dev_for(packed)
    p = _rows_2d(packed, dev, torch.uint8)
    n = p.shape[0]
    if p.shape[1] != packed_size(dim, bitwidth):
        raise FormatError("packed code block has the wrong size")
    out = torch.empty((n, dim), dtype=torch.uint8, device=dev)
    flags = new_flags(dev)
    _lib.check(_lib.lib().ds_unpack_code_rows(p.data_ptr(), n, dim, bitwidth, out.data_ptr(),
                                              flags.data_ptr(), _lib.stream_handle()),
               "unpack_code_rows")
    if int(flags.item()):
        raise FormatError("nonzero padding bits in packed codes")
    return like_input(out, packed)


# --- single-vector wrappers (quant.py:75-86, 118-131, 212-222, 398-412) -------

def _vector(vector) -> np.ndarray:
    x = np.asarray(vector, dtype=np.float32).reshape(-1)
    if x.size == 0:
        raise DataError("vector must be non-empty")
    if not np.isfinite(x).all():
        raise DataError("vector contains NaN or Inf")
    return x


def uniform_params(vector, bitwidth: int, mode: str = "asymmetric") -> QuantParams:
    x = _vector(vector)
    if mode == "asymmetric":
        lo, hi = row_minmax(x.reshape(1, -1))
        return QuantParams(bitwidth, float(lo[0]), float(hi[0]))
    if mode == "symmetric":
        m = float(np.abs(x).max())
        return QuantParams(bitwidth, -m, m)
    raise ConfigError(f"unknown mode {mode!r}")


def quantize(vector, params: QuantParams) -> QuantizedVector:
    x = _vector(vector).reshape(1, -1)
    codes = quantize_rows(x, np.float32([params.x_min]), np.float32([params.x_max]),
                          params.bitwidth)
    return QuantizedVector(params, codes[0])


def dequantize(qv: QuantizedVector) -> np.ndarray:
    codes = np.asarray(qv.codes, dtype=np.uint8).reshape(1, -1)
    return dequantize_rows(codes, np.float32([qv.params.x_min]), np.float32([qv.params.x_max]),
                           qv.params.bitwidth)[0]


def adaptive_params(vector, bitwidth: int, cfg: AdaptiveConfig | None = None) -> QuantParams:
    if cfg is None:
        cfg = default_adaptive_config(bitwidth)
        if cfg is None:
            return uniform_params(vector, bitwidth, "asymmetric")
    x = _vector(vector).reshape(1, -1)
    lo, hi = adaptive_params_rows(x, bitwidth, cfg)
    return QuantParams(bitwidth, float(lo[0]), float(hi[0]))


def pack_codes(codes, bitwidth: int) -> bytes:
    arr = np.asarray(codes, dtype=np.int64).reshape(1, -1)
    if arr.size and (arr.min() < 0 or arr.max() >= 2 ** bitwidth):
        raise DataError(f"code out of range for bitwidth {bitwidth}")
    return pack_code_rows(arr.astype(np.uint8), bitwidth).tobytes()


def unpack_codes(data: bytes, bitwidth: int, dim: int) -> np.ndarray:
    expected = packed_size(dim, bitwidth)
    if len(data) != expected:
        raise FormatError(f"expected {expected} packed bytes, got {len(data)}")
    packed = np.frombuffer(data, dtype=np.uint8).reshape(1, expected)
    return unpack_code_rows(packed, bitwidth, dim)[0]


def mean_l2_loss(original, reconstructed) -> float:
    """Mean over rows of the row-difference L2 (quant.py:225-231)."""
    a = np.atleast_2d(np.asarray(original, dtype=np.float64))
    b = np.atleast_2d(np.asarray(reconstructed, dtype=np.float64))
    if a.shape != b.shape:
        raise ShapeError(f"shape mismatch: {a.shape} vs {b.shape}")
    return float(np.linalg.norm(a - b, axis=1).mean())
