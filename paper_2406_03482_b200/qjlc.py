"""QJLC cache files from / into the device layout.

The reference serializes one `KeyCacheState` plus its value tokens per file
(`write_cache` / `read_cache`, pkg/src/qjl/kvcache.py:368-520):

    header  "<4sHHIIIIQHHQ" (48 B)  magic, version, flags, d, h, m_in, m_out, n,
                                    value_bits, 0, seed            (kvcache.py:371, :416-429)
    h outlier channels (u32), d channel magnitudes (f64)           (:431-432)
    n records: inlier words | f16 norm | outlier words | f16 norm |
               d one-byte codes | f32 zero | f32 scale             (:433-436, :472)

Here a `DeviceKeyCache` of U units maps to U such files (one unit = one
(batch, kv-head) pair = one reference `KeyCacheState`; the units share the seed,
so their sketches agree, and each has its own outlier profile).  The record
bytes are assembled / scattered on the GPU by `qjl_qjlc_export` /
`qjl_qjlc_import` (csrc/k_qjlc.cu); only the 48-byte header, the channels and
the magnitudes are host data.  Sign bytes are already the reference's (SURVEY
A.2) and norms already f16 (the file's own policy, kvcache.py:490), so the
conversion is exact both ways.  The file holds one zero/scale per token, so
the value cache must be in the reference's format: `value_layout="u8"` with
`value_group == d` (the group-32 P2/P2T fast-path layouts are not
representable and are rejected).
"""

from __future__ import annotations

import ctypes
import struct
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib

CACHE_MAGIC = b"QJLC"                     # kvcache.py:369
CACHE_VERSION = 1                         # kvcache.py:370
_HEADER = struct.Struct("<4sHHIIIIQHHQ")  # kvcache.py:371
HEADER_BYTES = _HEADER.size
FLAG_ORTHOGONALIZED = 1                   # kvcache.py:372


class FileFormatError(Exception):
    """A binary file failed magic/version/length validation (kvcache.py:34)."""


@dataclass(frozen=True)
class CacheHeader:
    """Decoded header fields of a cache file (kvcache.py:375-386)."""

    version: int
    d: int
    h: int
    m_in: int
    m_out: int
    n: int
    value_bits: int
    seed: int
    orthogonalized: bool


def _words(m: int) -> int:
    return (m + 63) // 64


def record_bytes(d: int, m_in: int, m_out: int) -> int:
    """Bytes per token record (kvcache.py:472)."""
    return 8 * _words(m_in) + 2 + 8 * _words(m_out) + 2 + d + 4 + 4


def pack_header(h: CacheHeader) -> bytes:
    return _HEADER.pack(CACHE_MAGIC, h.version, FLAG_ORTHOGONALIZED if h.orthogonalized else 0, h.d,
                        h.h, h.m_in, h.m_out, h.n, h.value_bits, 0, h.seed)


def parse_header(blob: bytes) -> CacheHeader:
    """Header of a whole file's bytes, with read_cache's checks (kvcache.py:447-464)."""
    if len(blob) < HEADER_BYTES:
        raise FileFormatError("cache file shorter than its header")
    magic, version, flags, d, h, m_in, m_out, n, value_bits, _, seed = _HEADER.unpack_from(blob)
    if magic != CACHE_MAGIC:
        raise FileFormatError(f"bad magic {magic!r}, expected {CACHE_MAGIC!r}")
    if version != CACHE_VERSION:
        raise FileFormatError(f"unsupported cache version {version}")
    expected = HEADER_BYTES + 4 * h + 8 * d + n * record_bytes(d, m_in, m_out)
    if len(blob) != expected:
        raise FileFormatError(
            f"cache payload length {len(blob)} does not match header (expected {expected})")
    return CacheHeader(version, d, h, m_in, m_out, n, value_bits, seed,
                       bool(flags & FLAG_ORTHOGONALIZED))


def profile_bytes(blob: bytes, hdr: CacheHeader) -> tuple[np.ndarray, np.ndarray]:
    """Outlier channels (u32) and per-channel magnitudes (f64) after the header."""
    ch = np.frombuffer(blob, "<u4", hdr.h, HEADER_BYTES).astype(np.int32)
    mags = np.frombuffer(blob, "<f8", hdr.d, HEADER_BYTES + 4 * hdr.h).copy()
    return ch, mags


def records_view(blob: bytes, hdr: CacheHeader) -> np.ndarray:
    """The n records of a file as a u8 [n, record_bytes] view."""
    off = HEADER_BYTES + 4 * hdr.h + 8 * hdr.d
    R = record_bytes(hdr.d, hdr.m_in, hdr.m_out)
    return np.frombuffer(blob, np.uint8, hdr.n * R, off).reshape(hdr.n, R)


def _stride(n: int, R: int) -> int:
    return (n * R + 15) // 16 * 16          # 16 B aligned unit spans (vector stores)


def _check_values(vd: _lib.ValueCacheDesc) -> None:
    if vd.layout != _lib.QJL_VLAYOUT_U8 or vd.group != vd.d:
        raise ValueError("QJLC files hold one zero/scale per token: the value cache must use "
                         "value_layout='u8' with value_group == d")


def export_records(keys: _lib.KeyCacheDesc, values: _lib.ValueCacheDesc, m_in: int, m_out: int,
                   n: int, row_offset: int = 0, out: torch.Tensor | None = None,
                   stream: int | None = None) -> tuple[torch.Tensor, int]:
    """Device records of rows [row_offset, row_offset + n) of every unit:
    u8 [units, stride], unit u's n records in out[u, :n * record_bytes]."""
    lib = _lib.load()
    _check_values(values)
    R = record_bytes(keys.d, m_in, m_out)
    stride = _stride(n, R)
    if out is None:
        out = torch.empty(keys.units, max(stride, 16), dtype=torch.uint8, device="cuda")
    st = torch.cuda.current_stream().cuda_stream if stream is None else stream
    _lib.check(lib.qjl_qjlc_export(ctypes.byref(keys), ctypes.byref(values), m_in, m_out, row_offset, n,
                                   out.data_ptr(), out.stride(0), st), "qjlc_export")
    return out, R


def import_records(records: torch.Tensor, n: int, m_in: int, m_out: int, keys: _lib.KeyCacheDesc,
                   values: _lib.ValueCacheDesc | None, row_offset: int = 0,
                   stream: int | None = None) -> None:
    """Scatter device records u8 [units, stride] into rows [row_offset, row_offset + n)."""
    lib = _lib.load()
    if values is not None:
        _check_values(values)
    st = torch.cuda.current_stream().cuda_stream if stream is None else stream
    _lib.check(lib.qjl_qjlc_import(records.data_ptr(), records.stride(0), n, m_in, m_out,
                                   ctypes.byref(keys), None if values is None else ctypes.byref(values),
                                   row_offset, st), "qjlc_import")


def save(cache, paths, magnitudes=None, n: int | None = None) -> None:
    """Write unit u of a `DeviceKeyCache` to paths[u] in the reference's format.

    magnitudes: [units, d] per-channel mean |k| of each unit's profile (default:
    the ones `cache.detect_outliers` computed)."""
    s = cache.shape
    paths = list(paths)
    if len(paths) != s.units:
        raise ValueError(f"{len(paths)} paths for {s.units} units")
    n = cache.n if n is None else n
    if n == 0:
        raise ValueError("refusing to serialize an empty cache")
    if n > cache.n_values:
        raise ValueError(f"value token count {cache.n_values} does not match cache length {n}")
    if magnitudes is None:
        magnitudes = getattr(cache, "magnitudes", None)
        if magnitudes is None:
            raise ValueError("no channel magnitudes: run detect_outliers or pass magnitudes=")
    mags = np.asarray(magnitudes.cpu() if torch.is_tensor(magnitudes) else magnitudes, np.float64)
    mags = mags.reshape(s.units, s.d)
    recs, R = export_records(cache.key_desc(), cache.value_desc(), s.m_in, s.m_out, n)
    host = torch.empty(recs.shape, dtype=torch.uint8, pin_memory=True)
    host.copy_(recs)
    chans = cache.channels[:, : s.h].cpu().numpy().astype("<u4")
    hdr = CacheHeader(CACHE_VERSION, s.d, s.h, s.m_in, s.m_out, n, cache.value_bits,
                      int(getattr(cache, "seed", 0)), bool(getattr(cache, "orthogonalized", False)))
    head = pack_header(hdr)
    hb = host.numpy()
    for u, p in enumerate(paths):
        with open(p, "wb") as f:
            f.write(head)
            f.write(chans[u].tobytes())
            f.write(mags[u].astype("<f8").tobytes())
            f.write(memoryview(hb[u, : n * R]))


def load(paths, key_dtype: torch.dtype = torch.float64, capacity: int | None = None):
    """Read U files written by `save` (or by the reference's write_cache) into one
    `DeviceKeyCache` of U units.  All files must share d, h, widths, n, value bits,
    seed and orthogonalization (they are units of one cache).  `key_dtype` picks the
    sketch operand (float64: the reference's own S, SIMT decode)."""
    from .device import DeviceKeyCache

    blobs = [open(p, "rb").read() for p in paths]
    if not blobs:
        raise ValueError("no cache files")
    hdrs = [parse_header(b) for b in blobs]
    h0 = hdrs[0]
    for h in hdrs[1:]:
        if (h.d, h.h, h.m_in, h.m_out, h.n, h.value_bits, h.seed, h.orthogonalized) != \
                (h0.d, h0.h, h0.m_in, h0.m_out, h0.n, h0.value_bits, h0.seed, h0.orthogonalized):
            raise ValueError("cache files disagree on shape, length, bit width or sketch seed")
    if h0.m_in % 32 or h0.m_out % 32:
        raise NotImplementedError("device caches hold sketch widths that are multiples of 32; "
                                  "use kvcache.read_cache for other widths")
    U, n, R = len(blobs), h0.n, record_bytes(h0.d, h0.m_in, h0.m_out)
    profs = [profile_bytes(b, h) for b, h in zip(blobs, hdrs)]
    chans = np.stack([c for c, _ in profs]) if h0.h else None
    cache = DeviceKeyCache.create(U, h0.d, h0.m_in, h=h0.h, m_out=h0.m_out if h0.h else 0,
                                  capacity=max(capacity or n, n, 1), seed=h0.seed,
                                  orthogonalize_sketches=h0.orthogonalized, channels=chans,
                                  key_dtype=key_dtype, value_layout="u8", value_bits=h0.value_bits,
                                  value_group=h0.d)
    stride = _stride(n, R)
    host = torch.zeros(U, max(stride, 16), dtype=torch.uint8, pin_memory=True)
    hb = host.numpy()
    for u, (b, h) in enumerate(zip(blobs, hdrs)):
        hb[u, : n * R] = records_view(b, h).reshape(-1)
    recs = host.to("cuda", non_blocking=True)
    import_records(recs, n, h0.m_in, h0.m_out, cache.key_desc(), cache.value_desc())
    cache.n = cache.n_values = n
    cache.magnitudes = torch.from_numpy(np.stack([m for _, m in profs])).to("cuda")
    torch.cuda.current_stream().synchronize()       # pinned staging buffer dies here
    return cache
