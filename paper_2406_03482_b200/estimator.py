"""Drop-in mirror of the reference estimator API (`pkg/src/qjl/estimator.py`),
executed on the B200 through the C ABI.  Same names, argument meaning, return
types and ValueError conditions; single-vector calls are correct but
launch-bound -- the batched path is `DeviceKeyCache`.

    quantize_key       estimator.py:110-124  -> qjl_quantize_keys (SIMT fp64 path)
    sketch_query       estimator.py:127-132  -> qjl_sketch_query
    packed_sign_dot    estimator.py:135-146  -> qjl_sign_dot_batch (n = 1)
    packed_sign_dot_batch estimator.py:149-170 -> qjl_sign_dot_batch
    estimate_inner_product estimator.py:173-186 -> device packed dot, exact zero rule
pack_signs / unpack_signs are host-side layout plumbing (estimator.py:49-71).
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .sketch import SketchMatrix

WORD_BITS = 64
ESTIMATOR_SCALE = math.sqrt(math.pi / 2)   # estimator.py:27
_WORD = np.dtype("<u8")


def _words_for(m: int) -> int:
    return (m + WORD_BITS - 1) // WORD_BITS


def _pad32(m: int) -> int:
    return (m + 31) // 32 * 32


def _bytes_to_words(b: np.ndarray, m: int) -> np.ndarray:
    """Device u8 rows (LSB-first) -> reference LE u64 words with zero padding."""
    nb = _words_for(m) * 8
    out = np.zeros(b.shape[:-1] + (nb,), np.uint8)
    k = min(nb, b.shape[-1])
    out[..., :k] = b[..., :k]
    # clear bits beyond m (padding must be zero, estimator.py:10-12)
    flat = out.reshape(-1, nb)
    if m % 8:
        flat[:, m // 8] &= np.uint8((1 << (m % 8)) - 1)
    flat[:, (m + 7) // 8:] = 0
    w = np.ascontiguousarray(out).view(_WORD)
    w.setflags(write=False)
    return w


def pack_signs(signs: np.ndarray) -> np.ndarray:
    """+/-1 vector -> LE u64 words, bit 1 == +1, LSB-first (estimator.py:49-59)."""
    signs = np.asarray(signs)
    if signs.ndim != 1 or signs.size == 0:
        raise ValueError("signs must be a non-empty 1-D vector")
    if not np.all(np.abs(signs) == 1):
        raise ValueError("signs must contain only +1 and -1")
    b = np.packbits(signs > 0, bitorder="little")
    return _bytes_to_words(b, signs.size)


def unpack_signs(words: np.ndarray, m: int) -> np.ndarray:
    """Inverse of pack_signs (estimator.py:62-71)."""
    words = np.asarray(words)
    if m < 1:
        raise ValueError(f"m must be positive, got {m}")
    if words.size != _words_for(m):
        raise ValueError(f"bit count mismatch: {words.size} words cannot hold exactly m={m} signs")
    raw = np.ascontiguousarray(words, dtype=_WORD).view(np.uint8)
    return np.where(np.unpackbits(raw, count=m, bitorder="little").astype(bool), 1, -1).astype(np.int8)


@dataclass(frozen=True, eq=False)
class QuantizedKey:
    """m packed sign bits + Euclidean norm (estimator.py:74-92)."""

    bits: np.ndarray
    norm: float
    m: int

    def __post_init__(self) -> None:
        if self.m < 0:
            raise ValueError("m must be non-negative")
        if self.bits.size != _words_for(self.m):
            raise ValueError("packed bit array length does not match m")
        if self.norm < 0:
            raise ValueError("key norm must be non-negative")


EMPTY_KEY = QuantizedKey(bits=np.empty(0, dtype=_WORD), norm=0.0, m=0)


@dataclass(frozen=True, eq=False)
class SketchedQuery:
    """Full-precision S @ q (estimator.py:98-107)."""

    values: np.ndarray
    source_dim: int

    @property
    def m(self) -> int:
        return int(self.values.shape[0])


# ----------------------------------------------------------------- helpers
def _dev() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("QJL device path needs CUDA (no CPU fallback)")
    return torch.device("cuda")


def _padded_sketch(sketch: SketchMatrix) -> torch.Tensor:
    m32 = _pad32(sketch.m)
    S = np.zeros((m32, sketch.d), np.float64)
    S[: sketch.m] = sketch.entries
    return torch.from_numpy(S).to(_dev())


def _quantize_rows(sketch: SketchMatrix, keys: np.ndarray):
    """Device quantize of keys [n, d] under one sketch -> (u8 rows, fp64 norms)."""
    lib = _lib.load()
    keys = np.asarray(keys, np.float64)
    n, d = keys.shape
    m32 = _pad32(sketch.m)
    dev = _dev()
    S = _padded_sketch(sketch)
    kt = torch.from_numpy(np.ascontiguousarray(keys)).to(dev)
    bits = torch.zeros(1, n, m32 // 8, dtype=torch.uint8, device=dev)
    norms = torch.zeros(1, n, dtype=torch.float16, device=dev)
    kd = _lib.KeyCacheDesc(bits.data_ptr(), None, norms.data_ptr(), None, n, 1, d, m32, 0, 0)
    sd = _lib.SketchDesc(S.data_ptr(), _lib.QJL_F64, 0, 0)
    _lib.check(lib.qjl_quantize_keys(kt.data_ptr(), _lib.QJL_F64, n, n * d, ctypes.byref(sd), None, 0,
                                     ctypes.byref(kd), 0, torch.cuda.current_stream().cuda_stream),
               "quantize_key")
    # norms at full working precision: the cache stores fp16, the
    # single-key API returns ||k||_2 exactly as the reference does.
    return bits[0].cpu().numpy(), np.sqrt(np.einsum("ij,ij->i", keys, keys))


def quantize_key(sketch: SketchMatrix, key: np.ndarray) -> QuantizedKey:
    """bits_i = (S k)_i >= 0, norm = ||k||_2 (estimator.py:110-124)."""
    key = np.asarray(key, dtype=np.float64)
    if key.shape != (sketch.d,):
        raise ValueError(f"key has shape {key.shape}, expected ({sketch.d},)")
    b, nrm = _quantize_rows(sketch, key[None, :])
    return QuantizedKey(bits=_bytes_to_words(b[0], sketch.m), norm=float(nrm[0]), m=sketch.m)


def sketch_query(sketch: SketchMatrix, query: np.ndarray) -> SketchedQuery:
    """S @ q on device (fp64 accumulation) (estimator.py:127-132)."""
    query = np.asarray(query, dtype=np.float64)
    if query.shape != (sketch.d,):
        raise ValueError(f"query has shape {query.shape}, expected ({sketch.d},)")
    lib = _lib.load()
    dev = _dev()
    S = torch.from_numpy(np.ascontiguousarray(sketch.entries, np.float64)).to(dev)
    q = torch.from_numpy(query).to(dev)
    out = torch.empty(sketch.m, dtype=torch.float64, device=dev)
    # the query-sketch kernel with fp64 accumulation and fp64 output (the drop-in returns
    # the full-precision projection, estimator.py:132)
    sd = _lib.SketchDesc(S.data_ptr(), _lib.QJL_F64, 0, 0)
    _lib.check(lib.qjl_sketch_query(q.data_ptr(), _lib.QJL_F64, 1, 1, sketch.d, ctypes.byref(sd), sketch.m,
                                    _lib.QJL_F64, out.data_ptr(), torch.cuda.current_stream().cuda_stream),
               "sketch_query")
    vals = out.cpu().numpy()
    vals.setflags(write=False)
    return SketchedQuery(values=vals, source_dim=sketch.d)


def packed_sign_dot_batch(word_rows: np.ndarray, m: int, values: np.ndarray,
                          chunk: int = 4096) -> np.ndarray:
    """Row-wise 2*sum_set(values) - sum(values), fp64 (estimator.py:149-170)."""
    lib = _lib.load()
    word_rows = np.ascontiguousarray(word_rows, dtype=_WORD)
    values = np.asarray(values, dtype=np.float64)
    n = word_rows.shape[0]
    if m == 0:
        return np.zeros(n)
    if n == 0:
        return np.empty(0)
    m32 = _pad32(m)
    rb = word_rows.view(np.uint8).reshape(n, -1)
    row_bytes = max(rb.shape[1], m32 // 8)
    row_bytes = (row_bytes + 3) // 4 * 4
    buf = np.zeros((n, row_bytes), np.uint8)
    buf[:, : rb.shape[1]] = rb
    # clear padding bits so the zero-padded values contribute nothing
    if m % 8:
        buf[:, m // 8] &= np.uint8((1 << (m % 8)) - 1)
    buf[:, (m + 7) // 8:] = 0
    v = np.zeros(m32, np.float64)
    v[:m] = values[:m]
    dev = _dev()
    bt = torch.from_numpy(buf).to(dev)
    vt = torch.from_numpy(v).to(dev)
    out = torch.empty(n, dtype=torch.float64, device=dev)
    _lib.check(lib.qjl_sign_dot_batch(bt.data_ptr(), n, m32, row_bytes, vt.data_ptr(), 1,
                                      out.data_ptr(), torch.cuda.current_stream().cuda_stream),
               "packed_sign_dot_batch")
    return out.cpu().numpy()


def packed_sign_dot(values: np.ndarray, words: np.ndarray, m: int) -> float:
    """<values, signs> from packed bits (estimator.py:135-146)."""
    if m == 0:
        return 0.0
    return float(packed_sign_dot_batch(np.asarray(words, _WORD)[None, :], m, values)[0])


def estimate_inner_product(query: SketchedQuery, key: QuantizedKey) -> float:
    """sqrt(pi/2)/m * ||k|| * <Sq, sign(Sk)>; zero norm / m -> exactly 0 (estimator.py:173-186)."""
    if query.m != key.m:
        raise ValueError(f"length mismatch: query has {query.m} coordinates, key has {key.m}")
    if key.m == 0 or key.norm == 0.0:
        return 0.0
    raw = packed_sign_dot(query.values, key.bits, key.m)
    return ESTIMATOR_SCALE / key.m * key.norm * raw
