"""CPU oracle for the QJL decode-time key path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline
leg / ``--impl reference`` arm may import this module.  The product package
(`paper_2406_03482_b200`) never calls it; the product fails loudly when its
CUDA library is missing.

What it is: a vectorised float64 numpy restatement of the reference's
hot-path algorithm (the reference is pure Python + numpy,
`/root/reference/pkg/src/qjl/`), one function per reference function, each
citing the file:line it follows.  The per-key reference loop is far too slow
at config scale (~30k keys/s), so whole (n, d) blocks are processed at once
with the same float64 arithmetic.

Parity pin: `tests/golden/make_golden.py` imports the real reference in the
build container and records its outputs (bits, norms, logits, scores, value
codes, decode outputs, outlier profiles) on seeded inputs into
`tests/golden/*.npz`; `tests/test_oracle_golden.py` checks this module
against every one of those vectors plus the SPEC.md known-answer examples.
Reference numpy dependency: numpy>=1.24 (`pkg/pyproject.toml:10`), run here
with numpy 2.3.5.

Storage policy: the device stores key norms and
value zero/scale constants as fp16; functions below take an explicit
``norm_dtype`` / ``const_dtype`` so the oracle sees the same rounded values
the reference's own `read_cache` would return (`kvcache.py:490`).
"""

from __future__ import annotations

import math

import numpy as np

# estimator.py:27
ESTIMATOR_SCALE = math.sqrt(math.pi / 2.0)
# kvcache.py:31
DEFAULT_OUTLIER_BITS_PER_CHANNEL = 8


# --------------------------------------------------------------------------
# bit packing: estimator.py:24-41 (LSB-first, little-endian u64 words)
# --------------------------------------------------------------------------
def words_for(m: int) -> int:
    """estimator.py:30-31."""
    return (m + 63) // 64


def pack_rows(flags: np.ndarray) -> np.ndarray:
    """Pack boolean rows (..., m) into u8 (..., 8*words_for(m)), LSB-first.

    Byte-identical to the reference's little-endian u64 words
    (estimator.py:34-41).
    """
    flags = np.asarray(flags, dtype=bool)
    m = flags.shape[-1]
    packed = np.packbits(flags, axis=-1, bitorder="little")
    nbytes = 8 * words_for(m)
    if packed.shape[-1] != nbytes:
        pad = np.zeros(flags.shape[:-1] + (nbytes - packed.shape[-1],), np.uint8)
        packed = np.concatenate([packed, pad], axis=-1)
    return packed


def unpack_rows(packed: np.ndarray, m: int) -> np.ndarray:
    """Inverse of pack_rows (estimator.py:44-46)."""
    return np.unpackbits(np.asarray(packed, np.uint8), axis=-1, count=m,
                         bitorder="little").astype(bool)


# --------------------------------------------------------------------------
# outlier profile: kvcache.py:66-123
# --------------------------------------------------------------------------
def detect_outliers(prompt_keys: np.ndarray, h: int):
    """Top-h channels by mean |k| (float64), ties -> lower index, sorted.

    kvcache.py:104-123 (mean at :116, lexsort at :118, sorted at :120).
    Returns (channels tuple, magnitudes float64[d]).
    """
    prompt_keys = np.asarray(prompt_keys, dtype=np.float64)
    if prompt_keys.ndim != 2 or prompt_keys.shape[0] == 0:
        raise ValueError("prompt keys must be a non-empty n x d matrix")
    d = prompt_keys.shape[1]
    if not 0 <= h <= d:
        raise ValueError(f"outlier count must be in [0, {d}], got {h}")
    mags = np.abs(prompt_keys).mean(axis=0)
    order = np.lexsort((np.arange(d), -mags))
    return tuple(sorted(int(c) for c in order[:h])), mags


def split_index(d: int, channels) -> tuple[np.ndarray, np.ndarray]:
    """(inlier ascending, outlier ascending) channel indices (kvcache.py:86-101)."""
    out_idx = np.asarray(sorted(channels), dtype=np.intp)
    mask = np.ones(d, dtype=bool)
    mask[out_idx] = False
    return np.flatnonzero(mask), out_idx


# --------------------------------------------------------------------------
# key quantization: estimator.py:110-124, kvcache.py:293-306
# --------------------------------------------------------------------------
def quantize_keys(S: np.ndarray | None, keys_part: np.ndarray):
    """Batched `quantize_key` over rows of keys_part (n, d_side).

    bits = pack(S @ k >= 0) (estimator.py:119-121), norm = ||k||_2 (:122).
    Empty side (S is None) -> no bits, norm 0 (EMPTY_KEY, estimator.py:95).
    Returns (bits u8[n, 8*words], norms float64[n], projections float64[n, m]).
    """
    keys_part = np.asarray(keys_part, dtype=np.float64)
    n = keys_part.shape[0]
    if S is None:
        return np.zeros((n, 0), np.uint8), np.zeros(n), np.zeros((n, 0))
    proj = keys_part @ np.asarray(S, np.float64).T
    # per-row norm exactly as np.linalg.norm does for a 1-D vector
    norms = np.sqrt(np.einsum("ij,ij->i", keys_part, keys_part))
    return pack_rows(proj >= 0), norms, proj


def append_keys(S_in, S_out, channels, keys: np.ndarray):
    """`KeyCacheState.append` for every row of keys (kvcache.py:293-306)."""
    keys = np.asarray(keys, dtype=np.float64)
    inl, outl = split_index(keys.shape[1], channels)
    b_in, n_in, p_in = quantize_keys(S_in, keys[:, inl])
    b_out, n_out, p_out = quantize_keys(S_out if len(outl) else None, keys[:, outl])
    return dict(bits_in=b_in, norm_in=n_in, proj_in=p_in,
                bits_out=b_out, norm_out=n_out, proj_out=p_out)


def fp16_round(x: np.ndarray) -> np.ndarray:
    """Storage policy: values round-trip through IEEE half (kvcache.py:430-432, :490)."""
    return np.asarray(x, np.float64).astype(np.float16).astype(np.float64)


# --------------------------------------------------------------------------
# score estimator: estimator.py:127-170, kvcache.py:311-337
# --------------------------------------------------------------------------
def sketch_query(S: np.ndarray, q: np.ndarray) -> np.ndarray:
    """S @ q in float64 (estimator.py:127-132)."""
    return np.asarray(S, np.float64) @ np.asarray(q, np.float64)


def packed_sign_dot_batch(bits: np.ndarray, m: int, values: np.ndarray) -> np.ndarray:
    """Row-wise 2*sum_{set}(values) - sum(values) (estimator.py:149-170)."""
    n = bits.shape[0]
    if m == 0:
        return np.zeros(n)
    values = np.asarray(values, np.float64)
    mask = unpack_rows(bits, m).astype(np.float64)
    return 2.0 * (mask @ values) - values.sum()


def side_logits(S, q_part, bits, norms) -> np.ndarray:
    """ESTIMATOR_SCALE / m * norms * raw (kvcache.py:311-320)."""
    if S is None:
        return np.zeros(bits.shape[0])
    m = S.shape[0]
    raw = packed_sign_dot_batch(bits, m, sketch_query(S, q_part))
    return ESTIMATOR_SCALE / m * np.asarray(norms, np.float64) * raw


def estimate_logits(S_in, S_out, channels, q, cache) -> np.ndarray:
    """Inlier + outlier side logits (kvcache.py:322-329)."""
    q = np.asarray(q, np.float64)
    inl, outl = split_index(q.shape[0], channels)
    if cache["bits_in"].shape[0] == 0:
        raise ValueError("cache is empty; append at least one key first")
    lg = side_logits(S_in, q[inl], cache["bits_in"], cache["norm_in"])
    if len(outl):
        lg = lg + side_logits(S_out, q[outl], cache["bits_out"], cache["norm_out"])
    return lg


def softmax(logits: np.ndarray) -> np.ndarray:
    """Max-subtracted float64 softmax (kvcache.py:38-44)."""
    z = np.asarray(logits, np.float64)
    w = np.exp(z - z.max())
    return w / w.sum()


# --------------------------------------------------------------------------
# values: kvcache.py:140-166, per group of `group` coordinates
# --------------------------------------------------------------------------
def quantize_values(values: np.ndarray, bits: int, group: int,
                    const_dtype: str | None = "f16"):
    """Token-wise affine quantization applied per `group`-wide slice.

    zero = min, scale = (max - min)/(2^b - 1), codes = clip(rint((v-zero)/scale))
    (kvcache.py:151-161, round-half-even via np.round); a constant slice gets
    scale 0 and zero codes (:154-156).  ``const_dtype="f16"`` rounds zero and
    scale to half precision AFTER computing the codes -- the device storage
    policy.  group == d reproduces the reference exactly.
    Returns (codes u8[n, d], zero f64[n, G], scale f64[n, G]).
    """
    v = np.asarray(values, np.float64)
    n, d = v.shape
    if d % group:
        raise ValueError("group must divide d")
    levels = (1 << bits) - 1
    g = v.reshape(n, d // group, group)
    zero = g.min(axis=2)
    spread = g.max(axis=2) - zero
    scale = np.where(spread == 0.0, 0.0, spread / levels)
    safe = np.where(spread == 0.0, 1.0, scale)
    codes = np.clip(np.round((g - zero[..., None]) / safe[..., None]), 0, levels)
    codes = np.where(spread[..., None] == 0.0, 0, codes).astype(np.uint8)
    if const_dtype == "f16":
        zero, scale = fp16_round(zero), fp16_round(scale)
    return codes.reshape(n, d), zero, scale


def dequantize_values(codes, zero, scale) -> np.ndarray:
    """zero + code * scale per group (kvcache.py:164-166)."""
    codes = np.asarray(codes, np.float64)
    n, d = codes.shape
    G = zero.shape[1]
    g = codes.reshape(n, G, d // G)
    return (zero[..., None] + g * scale[..., None]).reshape(n, d)


# --------------------------------------------------------------------------
# decode: attention.py:56-71
# --------------------------------------------------------------------------
def quantized_decode(S_in, S_out, channels, q, cache, values_deq, temperature=1.0):
    """weights = softmax(logits / T); output = weights @ values (attention.py:56-71)."""
    if temperature <= 0:
        raise ValueError(f"temperature must be positive, got {temperature}")
    logits = estimate_logits(S_in, S_out, channels, q, cache)
    w = softmax(logits / temperature)
    return w @ values_deq, w, logits


def decode_units(S_in, S_out, channels_per_unit, queries, caches, values_deq,
                 temperature=1.0):
    """GQA composition: every query head of a unit scores against that unit's
    state and aggregates its values.

    queries: [U, G, d]; caches: list of per-unit cache dicts; values_deq: [U, n, d].
    Returns out [U, G, d], logits [U, G, n].
    """
    U, G, d = queries.shape
    n = values_deq.shape[1]
    out = np.zeros((U, G, d))
    logits = np.zeros((U, G, n))
    for u in range(U):
        S_out_u = S_out if len(channels_per_unit[u]) else None
        for g in range(G):
            o, _, lg = quantized_decode(S_in, S_out_u, channels_per_unit[u],
                                        queries[u, g], caches[u], values_deq[u],
                                        temperature)
            out[u, g], logits[u, g] = o, lg
    return out, logits


# --------------------------------------------------------------------------
# QJLC cache files: kvcache.py:368-520 (write_cache / read_cache)
# --------------------------------------------------------------------------
QJLC_MAGIC = b"QJLC"                       # kvcache.py:369
QJLC_VERSION = 1                           # kvcache.py:370
QJLC_HEADER = "<4sHHIIIIQHHQ"              # kvcache.py:371 (48 bytes)
QJLC_FLAG_ORTHOGONALIZED = 1               # kvcache.py:372


def qjlc_record_bytes(d: int, m_in: int, m_out: int) -> int:
    """Bytes of one token record (kvcache.py:472): inlier words + f16 norm +
    outlier words + f16 norm + d one-byte codes + f32 zero + f32 scale."""
    return 8 * words_for(m_in) + 2 + 8 * words_for(m_out) + 2 + d + 4 + 4


def qjlc_encode(*, d, h, m_in, m_out, value_bits, seed, orthogonalized, channels, magnitudes,
                bits_in, norm_in, bits_out, norm_out, codes, zero, scale) -> bytes:
    """Serialize one unit exactly as write_cache does (kvcache.py:389-437).

    bits_*: u8 [n, >= ceil(m/8)] LSB-first sign bytes (columns past the side's
    8*words_for(m) bytes are ignored, missing ones are zero padding); norm_*:
    [n] (rounded to f16 here, :430/:432); codes u8 [n, d]; zero/scale [n]
    (rounded to f32, :434-435).  A side with m == 0 writes no words and a 0.0
    norm (EMPTY_KEY, estimator.py:95).
    """
    import struct
    n = int(np.asarray(codes).shape[0])
    if n == 0:
        raise ValueError("refusing to serialize an empty cache")             # :407-408
    flags = QJLC_FLAG_ORTHOGONALIZED if orthogonalized else 0
    head = struct.pack(QJLC_HEADER, QJLC_MAGIC, QJLC_VERSION, flags, d, h, m_in, m_out, n,
                       value_bits, 0, seed)                                  # :416-429

    def side(bits, norms, m):
        wb = 8 * words_for(m)
        out = np.zeros((n, wb), np.uint8)
        if m:
            b = np.asarray(bits, np.uint8)[:, :wb]
            out[:, : b.shape[1]] = b
        nv = np.zeros(n) if m == 0 else np.asarray(norms, np.float64)
        return out, nv.astype("<f2").view(np.uint8).reshape(n, 2)

    wi, ni = side(bits_in, norm_in, m_in)
    wo, no = side(bits_out, norm_out, m_out)
    z = np.asarray(zero, np.float64).astype("<f4").view(np.uint8).reshape(n, 4)
    s = np.asarray(scale, np.float64).astype("<f4").view(np.uint8).reshape(n, 4)
    rec = np.concatenate([wi, ni, wo, no, np.asarray(codes, np.uint8).reshape(n, d), z, s], axis=1)
    assert rec.shape[1] == qjlc_record_bytes(d, m_in, m_out)
    return (head + np.asarray(channels, "<u4").tobytes()
            + np.asarray(magnitudes, "<f8").tobytes() + rec.tobytes())


def qjlc_decode(blob: bytes) -> dict:
    """Parse a QJLC file as read_cache does (kvcache.py:440-520) into arrays.
    Raises ValueError where the reference raises FileFormatError (:452-464)."""
    import struct
    hs = struct.calcsize(QJLC_HEADER)
    if len(blob) < hs:
        raise ValueError("cache file shorter than its header")
    magic, version, flags, d, h, m_in, m_out, n, vbits, _, seed = struct.unpack_from(QJLC_HEADER, blob)
    if magic != QJLC_MAGIC:
        raise ValueError(f"bad magic {magic!r}")
    if version != QJLC_VERSION:
        raise ValueError(f"unsupported cache version {version}")
    R = qjlc_record_bytes(d, m_in, m_out)
    if len(blob) != hs + 4 * h + 8 * d + n * R:
        raise ValueError("cache payload length does not match header")
    off = hs
    channels = np.frombuffer(blob, "<u4", h, off).astype(np.int64)
    off += 4 * h
    mags = np.frombuffer(blob, "<f8", d, off).copy()
    off += 8 * d
    rec = np.frombuffer(blob, np.uint8, n * R, off).reshape(n, R)
    wi, wo = 8 * words_for(m_in), 8 * words_for(m_out)
    c = 0

    def take(k):
        nonlocal c
        r = rec[:, c:c + k]
        c += k
        return np.ascontiguousarray(r)

    bits_in = take(wi)
    norm_in = take(2).view("<f2")[:, 0].astype(np.float64)
    bits_out = take(wo)
    norm_out = take(2).view("<f2")[:, 0].astype(np.float64)
    codes = take(d)
    zero = take(4).view("<f4")[:, 0].astype(np.float64)
    scale = take(4).view("<f4")[:, 0].astype(np.float64)
    return dict(d=d, h=h, m_in=m_in, m_out=m_out, n=n, value_bits=vbits, seed=seed,
                orthogonalized=bool(flags & QJLC_FLAG_ORTHOGONALIZED), channels=channels,
                magnitudes=mags, bits_in=bits_in, norm_in=norm_in, bits_out=bits_out,
                norm_out=norm_out, codes=codes, zero=zero, scale=scale)
