"""B200-native checkpoint hot path of Check-N-Run (arXiv 2010.08679).

Drop-in for the hot-path names of the reference package `deltasnap`
(deltasnap/__init__.py:32-83): dirty-row tracking, the per-row codec, the
CNR1 payload layout, the shard payload writer and the restore scatter.  All
compute runs in hand-written sm_100a kernels (csrc/, C ABI in
include/deltasnap_cuda.h); there is no CPU fallback.
"""

from .errors import (
    BoundsError,
    ConfigError,
    DataError,
    DeltaSnapError,
    FormatError,
    IntegrityError,
    PreconditionError,
    ShapeError,
    StoreConflictError,
    StoreIOError,
)
from .tracker import DirtyBitmap, LookupStream, ModelTracker, TrackerView, lookup_width
from .quant import (
    AdaptiveConfig,
    QuantParams,
    QuantizedVector,
    VALID_BITWIDTHS,
    adaptive_params,
    adaptive_params_rows,
    default_adaptive_config,
    dequantize,
    dequantize_rows,
    mean_l2_loss,
    pack_code_rows,
    pack_codes,
    packed_size,
    quantize,
    quantize_rows,
    reconstruction_errors,
    uniform_params,
    unpack_code_rows,
    unpack_codes,
)
from .payload import (
    HEADER_SIZE,
    SECTION_MAGIC,
    TableSection,
    parse_shard_payload,
    serialize_section,
    serialize_shard_payload,
)
from .engine import (
    DeviceModelConfig,
    DeviceModelState,
    DeviceTable,
    IntervalSizes,
    ReaderPosition,
    RestoredRun,
    RestoredTables,
    ShardWriter,
    apply_payload,
    build_shard_payload,
    restore,
    restore_chain,
    stage_chain,
    state_digest,
)

__version__ = "0.1.0"
