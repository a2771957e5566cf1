"""Drop-in mirror of `pkg/src/qjl/kvcache.py` on the B200 device path.

Same names, constructor/method signatures, return types and ValueError
conditions as the reference; the state lives in a single-unit
`DeviceKeyCache` and every data-path operation runs as a CUDA kernel through
the C ABI (there is no CPU fallback):

    detect_outliers            kvcache.py:104-123  -> qjl_detect_outliers
    KeyCacheState.append       kvcache.py:293-306  -> qjl_quantize_keys (fp64 S, exact)
    KeyCacheState.estimate_logits  :322-329        -> qjl_scores
    KeyCacheState.estimate_scores  :331-337        -> qjl_scores + qjl_softmax_f64
    quantize_value             kvcache.py:140-161  -> qjl_quantize_values (U8 layout)
    write_cache / read_cache   kvcache.py:389-520  -> qjl_qjlc_export / qjl_qjlc_import

Storage policy (documented divergence, within the 1e-3 logit tolerance): key
norms are held at half precision, the reference's own serialization policy
(kvcache.py:430-432, :490), and value zero/scale at float32.  Sketch widths
that are not multiples of 32 are zero-padded on the device (padding bits are
cleared in the returned words, padded query coordinates are zero).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .device import DeviceKeyCache, _stream
from .estimator import EMPTY_KEY, QuantizedKey, _bytes_to_words, _pad32
from .sketch import SketchMatrix, derive_seed, generate_gaussian, orthogonalize

INLIER_STREAM = 0                      # kvcache.py:28
OUTLIER_STREAM = 1                     # kvcache.py:29
DEFAULT_OUTLIER_BITS_PER_CHANNEL = 8   # kvcache.py:31


from .qjlc import CACHE_MAGIC, CACHE_VERSION, CacheHeader, FileFormatError  # noqa: E402,F401
from . import qjlc as _qjlc  # noqa: E402


def _cuda() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("the QJL device path needs CUDA (no CPU fallback)")
    return torch.device("cuda")


def _softmax_rows(logits32: torch.Tensor, inv_t: float) -> np.ndarray:
    """fp64 softmax on the device of f32 logits [rows, n] * inv_t (kvcache.py:38-44)."""
    lib = _lib.load()
    rows, n = logits32.shape
    w = torch.empty(rows, n, dtype=torch.float64, device=logits32.device)
    _lib.check(lib.qjl_softmax_f64(logits32.data_ptr(), rows, n, float(inv_t), w.data_ptr(), _stream()),
               "softmax")
    return w.cpu().numpy()


def softmax(logits: np.ndarray) -> np.ndarray:
    """Numerically stable softmax, computed on the device in fp64 (kvcache.py:38-44)."""
    logits = np.asarray(logits, dtype=np.float64)
    t = torch.from_numpy(np.ascontiguousarray(logits.reshape(1, -1))).to(_cuda(), torch.float32)
    return _softmax_rows(t, 1.0)[0].reshape(logits.shape)


@dataclass(frozen=True, eq=False)
class ScoreVector:
    """Softmax-normalized attention weights (kvcache.py:47-63)."""

    weights: np.ndarray

    def __post_init__(self) -> None:
        if self.weights.ndim != 1 or self.weights.size == 0:
            raise ValueError("scores must be a non-empty 1-D vector")
        if np.any(self.weights < 0):
            raise ValueError("scores must be non-negative")
        if abs(float(self.weights.sum()) - 1.0) > 1e-6:
            raise ValueError("scores must sum to 1 within 1e-6")

    @property
    def n(self) -> int:
        return int(self.weights.shape[0])


@dataclass(frozen=True, eq=False)
class OutlierProfile:
    """Top-h channels by mean |k| over the prompt (kvcache.py:66-101)."""

    channels: tuple[int, ...]
    d: int
    channel_magnitudes: np.ndarray

    def __post_init__(self) -> None:
        if any(c < 0 or c >= self.d for c in self.channels):
            raise ValueError("outlier channels must lie in [0, d)")
        if list(self.channels) != sorted(set(self.channels)):
            raise ValueError("outlier channels must be sorted and unique")
        if self.channel_magnitudes.shape != (self.d,):
            raise ValueError("channel magnitudes must have one entry per channel")

    @property
    def h(self) -> int:
        return len(self.channels)

    @property
    def outlier_index(self) -> np.ndarray:
        return np.asarray(self.channels, dtype=np.intp)

    @property
    def inlier_index(self) -> np.ndarray:
        mask = np.ones(self.d, dtype=bool)
        mask[self.outlier_index] = False
        return np.flatnonzero(mask)

    def split(self, vector: np.ndarray) -> tuple[np.ndarray, np.ndarray]:
        vector = np.asarray(vector, dtype=np.float64)
        if vector.shape != (self.d,):
            raise ValueError(f"vector has shape {vector.shape}, expected ({self.d},)")
        return vector[self.inlier_index], vector[self.outlier_index]


def detect_outliers(prompt_keys: np.ndarray, h: int) -> OutlierProfile:
    """Top-h channels by mean |value| (fp64 on device), ties -> lower index (kvcache.py:104-123)."""
    lib = _lib.load()
    pk = np.asarray(prompt_keys, dtype=np.float64)
    if pk.ndim != 2 or pk.shape[0] == 0:
        raise ValueError("prompt keys must be a non-empty n x d matrix")
    n0, d = pk.shape
    if not 0 <= h <= d:
        raise ValueError(f"outlier count must be in [0, {d}], got {h}")
    dev = _cuda()
    kt = torch.from_numpy(np.ascontiguousarray(pk)).to(dev)
    ch = torch.zeros(max(h, 1), dtype=torch.int32, device=dev)
    mags = torch.zeros(d, dtype=torch.float64, device=dev)
    ws = torch.empty(max(int(lib.qjl_detect_workspace(1, n0, d)), 1), dtype=torch.uint8, device=dev)
    if h == 0:
        # magnitudes still come from the device reduction (h = 1 run, channel discarded)
        _lib.check(lib.qjl_detect_outliers(kt.data_ptr(), _lib.QJL_F64, 1, n0, d, n0 * d, 1,
                                           ch.data_ptr(), mags.data_ptr(), ws.data_ptr(), ws.numel(),
                                           _stream()), "detect_outliers")
        chans: tuple[int, ...] = ()
    else:
        _lib.check(lib.qjl_detect_outliers(kt.data_ptr(), _lib.QJL_F64, 1, n0, d, n0 * d, h,
                                           ch.data_ptr(), mags.data_ptr(), ws.data_ptr(), ws.numel(),
                                           _stream()), "detect_outliers")
        chans = tuple(int(c) for c in ch[:h].cpu().numpy())
    m = mags.cpu().numpy()
    m.setflags(write=False)
    return OutlierProfile(channels=chans, d=d, channel_magnitudes=m)


@dataclass(frozen=True, eq=False)
class QuantizedValueToken:
    """Per-token integer codes with an affine zero point and scale (kvcache.py:126-137)."""

    codes: np.ndarray
    zero: float
    scale: float
    bits: int

    @property
    def d(self) -> int:
        return int(self.codes.shape[0])


def quantize_value(values: np.ndarray, bits: int) -> QuantizedValueToken:
    """Token-wise affine quantization on the device (kvcache.py:140-161)."""
    if not 1 <= bits <= 8:
        raise ValueError(f"value bit width must be in [1, 8], got {bits}")
    values = np.asarray(values, dtype=np.float64)
    if values.ndim != 1 or values.size == 0:
        raise ValueError("value token must be a non-empty 1-D vector")
    lib = _lib.load()
    d = values.size
    dev = _cuda()
    vt = torch.from_numpy(np.ascontiguousarray(values)).to(dev)
    codes = torch.zeros(1, 1, d, dtype=torch.uint8, device=dev)
    zero = torch.zeros(1, 1, 1, dtype=torch.float32, device=dev)
    scale = torch.zeros(1, 1, 1, dtype=torch.float32, device=dev)
    vd = _lib.ValueCacheDesc(codes.data_ptr(), zero.data_ptr(), scale.data_ptr(), 1, 1, d, bits, d,
                             _lib.QJL_VLAYOUT_U8)
    _lib.check(lib.qjl_quantize_values(vt.data_ptr(), _lib.QJL_F64, 1, d, ctypes.byref(vd), 0, _stream()),
               "quantize_value")
    c = codes[0, 0].cpu().numpy().copy()
    c.setflags(write=False)
    return QuantizedValueToken(codes=c, zero=float(zero.item()), scale=float(scale.item()), bits=bits)


def dequantize_value(token: QuantizedValueToken) -> np.ndarray:
    """zero + code * scale (kvcache.py:164-166); layout helper, not on the decode path
    (the fused decode kernel dequantizes in registers)."""
    return token.zero + token.codes.astype(np.float64) * token.scale


@dataclass(frozen=True)
class MemoryReport:
    """Average storage bits per original floating-point number (kvcache.py:169-186)."""

    key_bits_per_fpn: float
    value_bits_per_fpn: float
    total_bits_per_fpn: float
    baseline_bits: float
    reduction_factor: float

    def as_dict(self) -> dict[str, float]:
        return dict(key_bits_per_fpn=self.key_bits_per_fpn, value_bits_per_fpn=self.value_bits_per_fpn,
                    total_bits_per_fpn=self.total_bits_per_fpn, baseline_bits=self.baseline_bits,
                    reduction_factor=self.reduction_factor)


class KeyCacheState:
    """Append-only stream of quantized keys under a fixed outlier profile
    (kvcache.py:189-365), stored on the device.  Single writer; readers see a
    consistent prefix (they pass the current length to the kernels)."""

    def __init__(self, profile: OutlierProfile, inlier_sketch: SketchMatrix | None,
                 outlier_sketch: SketchMatrix | None, seed: int = 0, orthogonalized: bool = False) -> None:
        d_in = profile.d - profile.h
        if (inlier_sketch is None) != (d_in == 0):
            raise ValueError("inlier sketch must be present exactly when d - h > 0")
        if (outlier_sketch is None) != (profile.h == 0):
            raise ValueError("outlier sketch must be present exactly when h > 0")
        if inlier_sketch is not None and inlier_sketch.d != d_in:
            raise ValueError(f"inlier sketch covers {inlier_sketch.d} channels, expected {d_in}")
        if outlier_sketch is not None and outlier_sketch.d != profile.h:
            raise ValueError(f"outlier sketch covers {outlier_sketch.d} channels, expected {profile.h}")
        if profile.h > 0 and d_in > 0:
            m_in, m_out = inlier_sketch.m, outlier_sketch.m
            if m_out * d_in < m_in * profile.h:
                raise ValueError("outlier bit rate below inlier bit rate: "
                                 f"m_out/h = {m_out}/{profile.h} < m_in/(d-h) = {m_in}/{d_in}")
        self.profile = profile
        self.inlier_sketch = inlier_sketch
        self.outlier_sketch = outlier_sketch
        self.seed = int(seed)
        self.orthogonalized = bool(orthogonalized)
        self._cap = 0
        self._dev: DeviceKeyCache | None = None
        self._n = 0
        # ||k_side||_2 at full precision, as quantize_key returns it (estimator.py:122); the
        # device keeps the fp16 copies its logits use (read_cache semantics, kvcache.py:490)
        self._norms = np.zeros((0, 2))
        self._grow(64)

    # ------------------------------------------------------------------ device
    def _padded(self, sk: SketchMatrix | None) -> np.ndarray | None:
        if sk is None:
            return None
        S = np.zeros((_pad32(sk.m), sk.d), np.float64)
        S[: sk.m] = sk.entries
        return S

    def _grow(self, need: int) -> None:
        cap = max(need, 2 * self._cap, 64)
        p = self.profile
        m_in = _pad32(self.m_in) if self.m_in else 0
        m_out = _pad32(self.m_out) if self.m_out else 0
        new = DeviceKeyCache(1, p.d, m_in, m_out, p.h, cap, key_dtype=torch.float64,
                             sketch_dtype=torch.float64, with_values=False, device=_cuda(),
                             validate_rate=False, tiled=False)   # rate already checked on the logical sizes
        if p.h:
            new.set_channels(np.asarray(p.channels, np.int32).reshape(1, p.h))
        new.set_sketches(self._padded(self.inlier_sketch), self._padded(self.outlier_sketch))
        if self._dev is not None and self._n:
            n = self._n
            new.bits_in[:, :n].copy_(self._dev.bits_in[:, :n])
            new.norm_in[:, :n].copy_(self._dev.norm_in[:, :n])
            if m_out:
                new.bits_out[:, :n].copy_(self._dev.bits_out[:, :n])
                new.norm_out[:, :n].copy_(self._dev.norm_out[:, :n])
        new.n = self._n
        self._dev, self._cap = new, new.shape.capacity

    @classmethod
    def create(cls, profile: OutlierProfile, m_in: int, m_out: int | None = None, seed: int = 0,
               orthogonalize_sketches: bool = True) -> "KeyCacheState":
        """Sub-sketches seeded derive_seed(seed, 0 / 1), m_out default 8*h (kvcache.py:234-267)."""
        h, d_in = profile.h, profile.d - profile.h
        if m_out is None:
            m_out = DEFAULT_OUTLIER_BITS_PER_CHANNEL * h

        def build(m: int, d: int, stream: int) -> SketchMatrix | None:
            if d == 0:
                return None
            sk = generate_gaussian(m, d, derive_seed(seed, stream))
            return orthogonalize(sk) if orthogonalize_sketches else sk

        return cls(profile=profile, inlier_sketch=build(m_in, d_in, INLIER_STREAM),
                   outlier_sketch=build(m_out, h, OUTLIER_STREAM), seed=seed,
                   orthogonalized=orthogonalize_sketches)

    @property
    def n(self) -> int:
        return self._n

    @property
    def d(self) -> int:
        return self.profile.d

    @property
    def h(self) -> int:
        return self.profile.h

    @property
    def m_in(self) -> int:
        return 0 if self.inlier_sketch is None else self.inlier_sketch.m

    @property
    def m_out(self) -> int:
        return 0 if self.outlier_sketch is None else self.outlier_sketch.m

    @property
    def device_cache(self) -> DeviceKeyCache:
        return self._dev

    @property
    def entries(self) -> tuple[tuple[QuantizedKey, QuantizedKey], ...]:
        """Materialize the (inlier, outlier) QuantizedKey pairs from the device."""
        n = self._n
        if n == 0:
            return ()
        c = self._dev
        bi = c.bits_in[0, :n].cpu().numpy()
        ni = self._norms[:n, 0]
        out = []
        bo = c.bits_out[0, :n].cpu().numpy() if self.m_out else None
        no = self._norms[:n, 1]
        for i in range(n):
            ki = QuantizedKey(bits=_bytes_to_words(bi[i], self.m_in), norm=float(ni[i]), m=self.m_in) \
                if self.m_in else EMPTY_KEY
            ko = QuantizedKey(bits=_bytes_to_words(bo[i], self.m_out), norm=float(no[i]), m=self.m_out) \
                if self.m_out else EMPTY_KEY
            out.append((ki, ko))
        return tuple(out)

    def append(self, key: np.ndarray) -> None:
        """Split by the profile, quantize each side, append (kvcache.py:293-306)."""
        key = np.asarray(key, dtype=np.float64)
        if key.shape != (self.d,):
            raise ValueError(f"vector has shape {key.shape}, expected ({self.d},)")
        self.extend(key[None, :])

    def extend(self, keys: np.ndarray) -> None:
        """Batched append of keys [t, d] in one launch (same result as t appends)."""
        keys = np.asarray(keys, dtype=np.float64)
        if keys.ndim != 2 or keys.shape[1] != self.d:
            raise ValueError(f"keys have shape {keys.shape}, expected (t, {self.d})")
        t = keys.shape[0]
        if self._n + t > self._cap:
            self._grow(self._n + t)
        kt = torch.from_numpy(np.ascontiguousarray(keys)).to(_cuda())[None]
        self._dev.n = self._n
        self._dev.append_keys(kt)
        p = self.profile
        inl, outl = p.inlier_index, p.outlier_index
        # per key exactly as quantize_key computes it (np.linalg.norm of the side vector)
        norms = np.array([[float(np.linalg.norm(k[inl])), float(np.linalg.norm(k[outl]))] for k in keys]
                         ).reshape(t, 2)
        self._norms = np.concatenate([self._norms[: self._n], norms])
        self._n += t
        self._clear_padding(self._n - t, self._n)

    def _clear_padding(self, a: int, b: int) -> None:
        # padded sketch rows project to 0 -> bit 1; the reference pads with 0 bits
        for bits, m in ((self._dev.bits_in, self.m_in), (self._dev.bits_out, self.m_out)):
            if bits is None or m == 0 or m % 32 == 0:
                continue
            if m % 8:
                bits[0, a:b, m // 8] &= (1 << (m % 8)) - 1
            bits[0, a:b, (m + 7) // 8:] = 0

    def _append_quantized(self, entry: tuple[QuantizedKey, QuantizedKey]) -> None:
        if self._n + 1 > self._cap:
            self._grow(self._n + 1)
        ki, ko = entry
        row = self._n
        for k, bits, norms, m in ((ki, self._dev.bits_in, self._dev.norm_in, self.m_in),
                                  (ko, self._dev.bits_out, self._dev.norm_out, self.m_out)):
            if m == 0:
                continue
            b = np.ascontiguousarray(k.bits, dtype="<u8").view(np.uint8)[: bits.shape[2]]
            bits[0, row, : b.size].copy_(torch.from_numpy(b.copy()))
            norms[0, row] = float(k.norm)
        self._norms = np.concatenate([self._norms[: self._n], [[float(ki.norm), float(ko.norm)]]])
        self._n += 1
        self._dev.n = self._n

    def _query_tensor(self, query: np.ndarray) -> torch.Tensor:
        q = np.array(query, dtype=np.float64)
        if q.shape != (self.d,):
            raise ValueError(f"vector has shape {q.shape}, expected ({self.d},)")
        # The device scales each side by sqrt(pi/2)/m_padded; logits are linear in q and
        # S_full keeps the sides on disjoint columns, so scaling the query's inlier /
        # outlier channels by m_padded/m restores the reference's sqrt(pi/2)/m exactly.
        if self.m_in and _pad32(self.m_in) != self.m_in:
            q[self.profile.inlier_index] *= _pad32(self.m_in) / self.m_in
        if self.m_out and _pad32(self.m_out) != self.m_out:
            q[self.profile.outlier_index] *= _pad32(self.m_out) / self.m_out
        return torch.from_numpy(np.ascontiguousarray(q)).to(_cuda())[None, None, :]

    def _logits32(self, query: np.ndarray) -> torch.Tensor:
        if self._n == 0:
            raise ValueError("cache is empty; append at least one key first")
        return self._dev.scores(self._query_tensor(query), n=self._n)[0]   # [1, n] f32

    def estimate_logits(self, query: np.ndarray) -> np.ndarray:
        """Per-token estimates <q, k_j>, inlier + outlier parts (kvcache.py:322-329)."""
        return self._logits32(query)[0].double().cpu().numpy()

    def estimate_scores(self, query: np.ndarray, temperature: float = 1.0) -> ScoreVector:
        """Softmax of logits / temperature (kvcache.py:331-337)."""
        if temperature <= 0:
            raise ValueError(f"temperature must be positive, got {temperature}")
        return ScoreVector(weights=_softmax_rows(self._logits32(query), 1.0 / temperature)[0])

    def memory_report(self, value_bits: int, norm_bits: int = 16, zero_bits: int = 16,
                      scale_bits: int = 16) -> MemoryReport:
        """Bits-per-FPN bookkeeping (kvcache.py:339-365)."""
        if self._n == 0:
            raise ValueError("memory report requires a non-empty cache")
        d = float(self.d)
        key_bits = (self.m_in + self.m_out + 2 * norm_bits) / d
        value_bits_per_fpn = value_bits + (zero_bits + scale_bits) / d
        total = (key_bits + value_bits_per_fpn) / 2.0
        return MemoryReport(key_bits, value_bits_per_fpn, total, 16.0, 16.0 / total)


def write_cache(path, state: KeyCacheState, value_tokens: list[QuantizedValueToken]) -> None:
    """Serialize a key-cache state and its value tokens (kvcache.py:389-437).

    The key records come straight from the state's device cache; the value tokens
    are staged as a one-unit U8 value cache, and `qjl_qjlc_export` assembles the
    record bytes on the GPU."""
    if state.n == 0:
        raise ValueError("refusing to serialize an empty cache")
    if len(value_tokens) != state.n:
        raise ValueError(
            f"value token count {len(value_tokens)} does not match cache length {state.n}")
    bits = value_tokens[0].bits
    if any(t.bits != bits or t.d != state.d for t in value_tokens):
        raise ValueError("value tokens must share one bit width and dimension")
    dev, n, d = _cuda(), state.n, state.d
    codes = torch.from_numpy(np.stack([np.asarray(t.codes, np.uint8) for t in value_tokens])).to(dev)
    zero = torch.tensor([t.zero for t in value_tokens], dtype=torch.float64).to(torch.float32).to(dev)
    scale = torch.tensor([t.scale for t in value_tokens], dtype=torch.float64).to(torch.float32).to(dev)
    vd = _lib.ValueCacheDesc(codes.data_ptr(), zero.data_ptr(), scale.data_ptr(), n, 1, d, bits, d,
                             _lib.QJL_VLAYOUT_U8)
    recs, R = _qjlc.export_records(state.device_cache.key_desc(), vd, state.m_in, state.m_out, n)
    hdr = CacheHeader(CACHE_VERSION, d, state.h, state.m_in, state.m_out, n, bits, state.seed,
                      state.orthogonalized)
    body = recs[0, : n * R].cpu().numpy()
    with open(path, "wb") as handle:
        handle.write(_qjlc.pack_header(hdr))
        handle.write(np.asarray(state.profile.channels, dtype="<u4").tobytes())
        handle.write(np.asarray(state.profile.channel_magnitudes, "<f8").tobytes())
        handle.write(body.tobytes())


def read_cache(path) -> tuple[KeyCacheState, list[QuantizedValueToken], CacheHeader]:
    """Load a cache file written by write_cache (kvcache.py:440-520).

    Sketches are regenerated from the header; the key records are scattered into
    the state's device cache by `qjl_qjlc_import`; value tokens are returned as
    host objects with f32-valued zero/scale, as the reference returns them."""
    with open(path, "rb") as handle:
        blob = handle.read()
    hdr = _qjlc.parse_header(blob)
    channels, mags = _qjlc.profile_bytes(blob, hdr)
    mags.setflags(write=False)
    profile = OutlierProfile(channels=tuple(int(c) for c in channels), d=hdr.d, channel_magnitudes=mags)
    state = KeyCacheState.create(profile, m_in=hdr.m_in, m_out=hdr.m_out if hdr.h > 0 else 0,
                                 seed=hdr.seed, orthogonalize_sketches=hdr.orthogonalized)
    n = hdr.n
    recs_np = _qjlc.records_view(blob, hdr)
    if n:
        if n > state._cap:
            state._grow(n)
        recs = torch.from_numpy(np.array(recs_np).reshape(1, -1)).to(_cuda())
        _qjlc.import_records(recs, n, state.m_in, state.m_out, state.device_cache.key_desc(), None)
        state._n = n
        dc = state.device_cache
        dc.n = n
        # the file's f16 norms are the entries' norms (read_cache semantics, kvcache.py:490)
        ni = dc.norm_in[0, :n].double().cpu().numpy()
        no = dc.norm_out[0, :n].double().cpu().numpy() if state.m_out else np.zeros(n)
        state._norms = np.stack([ni, no], axis=1)
    R = recs_np.shape[1]
    c0 = R - hdr.d - 8
    codes = np.ascontiguousarray(recs_np[:, c0:c0 + hdr.d])
    zero = np.ascontiguousarray(recs_np[:, R - 8:R - 4]).view("<f4")[:, 0].astype(np.float64)
    scale = np.ascontiguousarray(recs_np[:, R - 4:]).view("<f4")[:, 0].astype(np.float64)
    tokens = []
    for i in range(n):
        c = codes[i].copy()
        c.setflags(write=False)
        tokens.append(QuantizedValueToken(codes=c, zero=float(zero[i]), scale=float(scale[i]),
                                          bits=hdr.value_bits))
    return state, tokens, hdr
