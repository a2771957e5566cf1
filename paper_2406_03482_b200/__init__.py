"""paper_2406_03482_b200 -- B200-native (sm_100a) QJL decode-time key path.

Drop-in for the reference package's quantizer / estimator / key-cache /
quantized-decode API (`pkg/src/qjl/__init__.py:10-93`, hot-path names only,
SURVEY 8(b)), executed by hand-written CUDA kernels through the C ABI in
include/qjl_b200.h, plus the batched device-resident `DeviceKeyCache` used for
serving-scale work.  Importing the package does not touch the GPU; calls that
need the device fail loudly when the library or a CUDA device is missing.
"""

from .attention import DecodeResult, quantized_decode
from .device import DeviceKeyCache, pack_codes, unpack_codes
from .distributed import UnitShard, gather_units, shard_of, shard_units
from .estimator import (
    EMPTY_KEY,
    ESTIMATOR_SCALE,
    QuantizedKey,
    SketchedQuery,
    estimate_inner_product,
    pack_signs,
    packed_sign_dot,
    packed_sign_dot_batch,
    quantize_key,
    sketch_query,
    unpack_signs,
)
from .kvcache import (
    CACHE_MAGIC,
    CACHE_VERSION,
    CacheHeader,
    FileFormatError,
    KeyCacheState,
    MemoryReport,
    OutlierProfile,
    QuantizedValueToken,
    ScoreVector,
    dequantize_value,
    detect_outliers,
    quantize_value,
    read_cache,
    softmax,
    write_cache,
)
from .sketch import SketchMatrix, derive_seed, generate_gaussian, orthogonalize, rng_from_seed

__version__ = "0.1.0"

__all__ = [
    "CACHE_MAGIC", "CACHE_VERSION", "CacheHeader", "FileFormatError", "read_cache", "write_cache",
    "DecodeResult", "DeviceKeyCache", "EMPTY_KEY", "ESTIMATOR_SCALE", "KeyCacheState", "MemoryReport",
    "OutlierProfile", "QuantizedKey", "QuantizedValueToken", "ScoreVector", "SketchMatrix",
    "SketchedQuery", "UnitShard", "dequantize_value", "derive_seed", "detect_outliers",
    "estimate_inner_product", "gather_units", "generate_gaussian", "orthogonalize", "pack_codes",
    "unpack_codes", "pack_signs", "packed_sign_dot", "packed_sign_dot_batch", "quantize_key",
    "quantize_value", "quantized_decode", "rng_from_seed", "shard_of", "shard_units",
    "sketch_query", "softmax", "unpack_signs",
]
