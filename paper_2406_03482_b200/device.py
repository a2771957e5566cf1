"""Batched, device-resident QJL cache over U units (one unit = one (batch,
kv-head) pair).  This is the B200 hot path behind the reference API:

    reference (per key / per query, pkg/src/qjl/kvcache.py)   here (per launch, all units)
    KeyCacheState.create              :234-267                 DeviceKeyCache.create / set_sketches
    detect_outliers                   :104-123                 DeviceKeyCache.detect_outliers
    detect_outliers + create + append (fused, F2)              DeviceKeyCache.prefill
    KeyCacheState.append              :293-306                 DeviceKeyCache.append_keys      (K1)
    quantize_value                    :140-161                 DeviceKeyCache.append_values
    KeyCacheState.estimate_logits     :322-329                 DeviceKeyCache.scores            (K2)
    quantized_decode (attention.py:56-71)                      DeviceKeyCache.decode         (K2+K3)

All device memory is owned here as torch tensors; the C library allocates
nothing.  Calls are ordered on torch's current stream.  Readers pass the
current prefix length n, so a reader launched before an append sees the
consistent prefix (kvcache.py:189-196).
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .sketch import derive_seed, generate_gaussian, orthogonalize, round_to_operand

INLIER_STREAM, OUTLIER_STREAM = 0, 1          # kvcache.py:28-29
DEFAULT_OUTLIER_BITS_PER_CHANNEL = 8          # kvcache.py:31

_TORCH2QJL = {torch.float32: _lib.QJL_F32, torch.float16: _lib.QJL_F16,
              torch.bfloat16: _lib.QJL_BF16, torch.float64: _lib.QJL_F64}
_NAME2TORCH = {"f32": torch.float32, "f16": torch.float16, "bf16": torch.bfloat16,
               "f64": torch.float64}
_TORCH2NAME = {v: k for k, v in _NAME2TORCH.items()}


def operand_dtype_for(key_dtype: torch.dtype) -> torch.dtype:
    """Sketch operand dtype (SURVEY parity decision 1): bf16 keys -> bf16 S and
    fp16 keys -> fp16 S (tensor-core path); fp32/fp64 keys -> fp64 S (SIMT fp64
    path, which is then exact against the reference's own float64 S)."""
    return {torch.bfloat16: torch.bfloat16, torch.float16: torch.float16}.get(key_dtype,
                                                                             torch.float64)


def _ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()


def _stream() -> int:
    return torch.cuda.current_stream().cuda_stream


@dataclass
class CacheShape:
    units: int
    d: int
    m_in: int
    m_out: int
    h: int
    capacity: int


class DeviceKeyCache:
    """Packed QJL key cache + 2-bit (or u8) value cache for `units` units."""

    def __init__(self, units: int, d: int, m_in: int, m_out: int, h: int, capacity: int, *,
                 key_dtype: torch.dtype = torch.bfloat16, value_bits: int = 2,
                 value_group: int = 32, value_layout: str = "p2t", with_values: bool = True,
                 sketch_dtype: torch.dtype | None = None, device: str | torch.device = "cuda",
                 validate_rate: bool = True):
        self.lib = _lib.load()
        if not torch.cuda.is_available():
            raise RuntimeError("DeviceKeyCache needs a CUDA device (no CPU fallback)")
        if units < 1 or capacity < 1:
            raise ValueError("units and capacity must be >= 1")
        if not 0 <= h <= d:
            raise ValueError(f"outlier count must be in [0, {d}], got {h}")
        if (m_out > 0) != (h > 0):
            raise ValueError("outlier sketch must be present exactly when h > 0")
        if (m_in > 0) != (d - h > 0):
            raise ValueError("inlier sketch must be present exactly when d - h > 0")
        if validate_rate and h > 0 and d - h > 0 and m_out * (d - h) < m_in * h:
            raise ValueError("outlier bit rate below inlier bit rate: "
                             f"m_out/h = {m_out}/{h} < m_in/(d-h) = {m_in}/{d - h}")
        self.device = torch.device(device)
        # rows are padded to whole 128-token tiles: the tensor-core decode streams
        # full tiles with bulk copies and masks tokens >= n
        capacity = (capacity + 127) // 128 * 128
        self.shape = CacheShape(units, d, m_in, m_out, h, capacity)
        self.key_dtype = key_dtype
        self.sketch_dtype = sketch_dtype or operand_dtype_for(key_dtype)
        dev = self.device
        self.bits_in = torch.zeros(units, capacity, max(m_in, 8) // 8, dtype=torch.uint8, device=dev)
        self.norm_in = torch.zeros(units, capacity, dtype=torch.float16, device=dev)
        self.bits_out = (torch.zeros(units, capacity, m_out // 8, dtype=torch.uint8, device=dev)
                         if m_out else None)
        self.norm_out = torch.zeros(units, capacity, dtype=torch.float16, device=dev) if m_out else None
        self.channels = torch.zeros(units, max(h, 1), dtype=torch.int32, device=dev)
        self.s_full: torch.Tensor | None = None
        self.n = 0
        self.value_layout = value_layout
        self.with_values = with_values
        self.value_bits, self.value_group = value_bits, value_group
        if with_values:
            G = d // value_group
            if value_layout in ("p2", "p2t"):
                if not (d == 128 and value_bits == 2 and value_group == 32):
                    raise ValueError(f"{value_layout} value layout is 2-bit, group 32, d = 128")
                self.v_codes = torch.zeros(units, capacity, d // 4, dtype=torch.uint8, device=dev)
                self.v_zero = torch.zeros(units, capacity, G, dtype=torch.float16, device=dev)
                self.v_scale = torch.zeros(units, capacity, G, dtype=torch.float16, device=dev)
            elif value_layout == "u8":
                self.v_codes = torch.zeros(units, capacity, d, dtype=torch.uint8, device=dev)
                self.v_zero = torch.zeros(units, capacity, G, dtype=torch.float32, device=dev)
                self.v_scale = torch.zeros(units, capacity, G, dtype=torch.float32, device=dev)
            else:
                raise ValueError(f"unknown value layout {value_layout!r}")
        self.n_values = 0
        self._ws: torch.Tensor | None = None

    # ------------------------------------------------------------ descriptors
    def key_desc(self) -> _lib.KeyCacheDesc:
        s = self.shape
        return _lib.KeyCacheDesc(_ptr(self.bits_in), _ptr(self.bits_out), _ptr(self.norm_in),
                                 _ptr(self.norm_out), s.capacity, s.units, s.d, s.m_in, s.m_out)

    def value_desc(self) -> _lib.ValueCacheDesc:
        s = self.shape
        layout = {"p2": _lib.QJL_VLAYOUT_P2, "p2t": _lib.QJL_VLAYOUT_P2T}.get(self.value_layout,
                                                                             _lib.QJL_VLAYOUT_U8)
        return _lib.ValueCacheDesc(_ptr(self.v_codes), _ptr(self.v_zero), _ptr(self.v_scale),
                                   s.capacity, s.units, s.d, self.value_bits, self.value_group,
                                   layout)

    def sketch_desc(self) -> _lib.SketchDesc:
        if self.s_full is None:
            raise ValueError("sketches not set: call set_sketches() or create()")
        s = self.shape
        return _lib.SketchDesc(_ptr(self.s_full), _TORCH2QJL[self.sketch_dtype], 0,
                               (s.m_in + s.m_out) * s.d)

    def set_unit_sketches(self, s_full: torch.Tensor) -> None:
        """Give every unit its own zero-padded S_full [units, m_in + m_out, d] (operand
        dtype, on the device) -- e.g. one independent sketch per statistical trial."""
        s = self.shape
        if tuple(s_full.shape) != (s.units, s.m_in + s.m_out, s.d) or s_full.dtype != self.sketch_dtype:
            raise ValueError(f"per-unit sketches must be {self.sketch_dtype} "
                             f"[{s.units}, {s.m_in + s.m_out}, {s.d}], got {s_full.dtype} {tuple(s_full.shape)}")
        self.s_full = s_full.contiguous()

    def workspace(self, nbytes: int) -> torch.Tensor:
        if self._ws is None or self._ws.numel() < nbytes:
            self._ws = torch.empty(max(nbytes, 1), dtype=torch.uint8, device=self.device)
        return self._ws

    # ------------------------------------------------------------- profile/S
    def detect_outliers(self, prompt_keys: torch.Tensor) -> torch.Tensor:
        """Per-unit outlier channels from prompt keys [U, n0, d] (kvcache.py:104-123)."""
        s = self.shape
        pk = prompt_keys.contiguous()
        if pk.dim() != 3 or pk.shape[0] != s.units or pk.shape[2] != s.d or pk.shape[1] == 0:
            raise ValueError("prompt keys must be a non-empty [units, n0, d] tensor")
        mags = torch.empty(s.units, s.d, dtype=torch.float64, device=self.device)
        if s.h == 0:
            return self.channels[:, :0]
        _lib.check(self.lib.qjl_detect_outliers(pk.data_ptr(), _TORCH2QJL[pk.dtype], s.units,
                                                pk.shape[1], s.d, pk.shape[1] * s.d, s.h,
                                                self.channels.data_ptr(), mags.data_ptr(),
                                                _stream()), "detect_outliers")
        self.magnitudes = mags
        return self.channels

    def set_channels(self, channels) -> None:
        s = self.shape
        ch = torch.as_tensor(np.asarray(channels, dtype=np.int32).reshape(s.units, s.h))
        self.channels[:, : s.h].copy_(ch.to(self.device))

    def set_sketches(self, S_in: np.ndarray | None, S_out: np.ndarray | None) -> None:
        """Upload S_in [m_in, d-h] and S_out [m_out, h] (float64 host arrays, shared by
        all units) and build each unit's zero-padded S_full in the operand dtype."""
        s = self.shape
        dev = self.device
        sin = None if S_in is None else torch.as_tensor(np.ascontiguousarray(S_in, np.float64)).to(dev)
        sout = None if S_out is None else torch.as_tensor(np.ascontiguousarray(S_out, np.float64)).to(dev)
        if sin is not None and tuple(sin.shape) != (s.m_in, s.d - s.h):
            raise ValueError(f"inlier sketch covers {tuple(sin.shape)}, expected ({s.m_in}, {s.d - s.h})")
        if sout is not None and tuple(sout.shape) != (s.m_out, s.h):
            raise ValueError(f"outlier sketch covers {tuple(sout.shape)}, expected ({s.m_out}, {s.h})")
        self.s_full = torch.empty(s.units, s.m_in + s.m_out, s.d, dtype=self.sketch_dtype, device=dev)
        _lib.check(self.lib.qjl_build_sketch(_ptr(sin), _ptr(sout), s.m_in, s.m_out, s.d, s.h,
                                             self.channels.data_ptr(), s.units,
                                             _TORCH2QJL[self.sketch_dtype], self.s_full.data_ptr(),
                                             _stream()), "build_sketch")
        self._sketch_keepalive = (sin, sout)

    def prefill(self, prompt_keys: torch.Tensor, values: torch.Tensor | None = None) -> None:
        """Fused prompt profile + append: `qjl_prefill_profile` detects each
        unit's outlier channels and builds its zero-padded S_full in one pass over the prompt
        (kvcache.py:104-123, :234-267), then K1 quantizes the prompt into rows [n, n + n0)
        (kvcache.py:293-306) and the values, if given, are quantized alongside."""
        s = self.shape
        pk = prompt_keys.contiguous()
        if pk.dim() != 3 or pk.shape[0] != s.units or pk.shape[2] != s.d or pk.shape[1] == 0:
            raise ValueError("prompt keys must be a non-empty [units, n0, d] tensor")
        if getattr(self, "S_in_host", None) is None and getattr(self, "S_out_host", None) is None:
            raise ValueError("no host sketches: build the cache with DeviceKeyCache.create")
        dev = self.device
        if getattr(self, "_sk_op", None) is None:
            # S_in / S_out in the operand dtype (exact: the host copies are operand-rounded)
            self._sk_op = tuple(None if S is None else
                                torch.as_tensor(np.ascontiguousarray(S, np.float64)).to(dev, self.sketch_dtype)
                                for S in (self.S_in_host, self.S_out_host))
        sin, sout = self._sk_op
        if self.s_full is None:
            self.s_full = torch.empty(s.units, s.m_in + s.m_out, s.d, dtype=self.sketch_dtype, device=dev)
        mags = torch.empty(s.units, s.d, dtype=torch.float64, device=dev)
        _lib.check(self.lib.qjl_prefill_profile(pk.data_ptr(), _TORCH2QJL[pk.dtype], s.units, pk.shape[1],
                                                s.d, pk.shape[1] * s.d, s.h, _ptr(sin), _ptr(sout),
                                                s.m_in, s.m_out, _TORCH2QJL[self.sketch_dtype],
                                                self.channels.data_ptr(), mags.data_ptr(),
                                                self.s_full.data_ptr(), _stream()), "prefill_profile")
        self.magnitudes = mags
        self.append(pk, values)

    @staticmethod
    def make_sketches(d: int, h: int, m_in: int, m_out: int, seed: int = 0,
                      orthogonalize_sketches: bool = True, operand: str | None = None):
        """S_in, S_out exactly as KeyCacheState.create draws them (kvcache.py:234-267),
        optionally rounded to the device operand dtype (and returned as float64)."""
        def build(m, dd, stream):
            if dd == 0 or m == 0:
                return None
            sk = generate_gaussian(m, dd, derive_seed(seed, stream))
            e = (orthogonalize(sk) if orthogonalize_sketches else sk).entries
            return round_to_operand(e, operand) if operand else np.array(e)
        return build(m_in, d - h, INLIER_STREAM), build(m_out, h, OUTLIER_STREAM)

    # ------------------------------------------------------------- appends
    def append_keys(self, keys: torch.Tensor) -> None:
        """K1: quantize keys [U, t, d] into rows [n, n + t) (kvcache.py:293-306)."""
        s = self.shape
        k = keys.contiguous()
        if k.dim() != 3 or k.shape[0] != s.units or k.shape[2] != s.d:
            raise ValueError(f"keys have shape {tuple(k.shape)}, expected ({s.units}, t, {s.d})")
        t = k.shape[1]
        if self.n + t > s.capacity:
            raise ValueError(f"cache capacity {s.capacity} exceeded")
        kd = self.key_desc()
        sd = self.sketch_desc()
        _lib.check(self.lib.qjl_quantize_keys(k.data_ptr(), _TORCH2QJL[k.dtype], t, t * s.d,
                                              ctypes.byref(sd), self.channels.data_ptr(), s.h,
                                              ctypes.byref(kd), self.n, _stream()), "quantize_keys")
        self.n += t

    def append_values(self, values: torch.Tensor) -> None:
        """Quantize values [U, t, d] into rows [n_values, n_values + t) (kvcache.py:140-161)."""
        s = self.shape
        v = values.contiguous()
        if v.dim() != 3 or v.shape[0] != s.units or v.shape[2] != s.d:
            raise ValueError(f"values have shape {tuple(v.shape)}, expected ({s.units}, t, {s.d})")
        t = v.shape[1]
        if self.n_values + t > s.capacity:
            raise ValueError(f"cache capacity {s.capacity} exceeded")
        vd = self.value_desc()
        _lib.check(self.lib.qjl_quantize_values(v.data_ptr(), _TORCH2QJL[v.dtype], t, t * s.d,
                                                ctypes.byref(vd), self.n_values, _stream()),
                   "quantize_values")
        self.n_values += t

    def append(self, keys: torch.Tensor, values: torch.Tensor | None = None) -> None:
        self.append_keys(keys)
        if values is not None:
            self.append_values(values)

    # ------------------------------------------------------------- readers
    def _check_q(self, q: torch.Tensor) -> torch.Tensor:
        s = self.shape
        q = q.contiguous()
        if q.dim() != 3 or q.shape[0] != s.units or q.shape[2] != s.d:
            raise ValueError(f"queries have shape {tuple(q.shape)}, expected ({s.units}, G, {s.d})")
        return q

    def sketch_query(self, q: torch.Tensor) -> torch.Tensor:
        """S_full @ q for q [U, G, d] -> [U, G, m_in + m_out] f32 (estimator.py:127-132)."""
        s = self.shape
        q = self._check_q(q)
        out = torch.empty(s.units, q.shape[1], s.m_in + s.m_out, dtype=torch.float32, device=self.device)
        sd = self.sketch_desc()
        _lib.check(self.lib.qjl_sketch_query(q.data_ptr(), _TORCH2QJL[q.dtype], s.units, q.shape[1],
                                             s.d, ctypes.byref(sd), s.m_in + s.m_out,
                                             out.data_ptr(), _stream()), "sketch_query")
        return out

    def scores(self, q: torch.Tensor, n: int | None = None, out: torch.Tensor | None = None) -> torch.Tensor:
        """K2: logits [U, G, n] f32 (kvcache.py:311-329)."""
        s = self.shape
        q = self._check_q(q)
        n = self.n if n is None else n
        G = q.shape[1]
        if out is None:
            out = torch.empty(s.units, G, max(n, 1), dtype=torch.float32, device=self.device)
        ws_b = self.lib.qjl_scores_workspace(s.units, G, s.m_in + s.m_out)
        ws = self.workspace(ws_b)
        kd, sd = self.key_desc(), self.sketch_desc()
        _lib.check(self.lib.qjl_scores(ctypes.byref(kd), n, q.data_ptr(), _TORCH2QJL[q.dtype], G,
                                       ctypes.byref(sd), out.data_ptr(), ws.data_ptr(), ws.numel(),
                                       _stream()), "scores")
        return out

    def decode_workspace_bytes(self, G: int, n: int | None = None) -> int:
        n = self.n if n is None else n
        kd, vd = self.key_desc(), self.value_desc()
        return int(self.lib.qjl_decode_workspace(ctypes.byref(kd), ctypes.byref(vd), n, G))

    def decode(self, q: torch.Tensor, temperature: float = 1.0, n: int | None = None,
               out: torch.Tensor | None = None, lse: torch.Tensor | None = None) -> torch.Tensor:
        """K2+K3: softmax(logits / T) @ V per query head -> [U, G, d] f32 (attention.py:56-71)."""
        if temperature <= 0:
            raise ValueError(f"temperature must be positive, got {temperature}")
        if not self.with_values:
            raise ValueError("cache was created without values")
        s = self.shape
        q = self._check_q(q)
        n = self.n if n is None else n
        if n > self.n_values:
            raise ValueError(f"cache holds {self.n} keys but {self.n_values} value tokens")
        G = q.shape[1]
        if out is None:
            out = torch.empty(s.units, G, s.d, dtype=torch.float32, device=self.device)
        kd, vd, sd = self.key_desc(), self.value_desc(), self.sketch_desc()
        ws_b = int(self.lib.qjl_decode_workspace(ctypes.byref(kd), ctypes.byref(vd), n, G))
        ws = self.workspace(ws_b)
        _lib.check(self.lib.qjl_decode(ctypes.byref(kd), ctypes.byref(vd), n, q.data_ptr(),
                                       _TORCH2QJL[q.dtype], G, ctypes.byref(sd),
                                       1.0 / float(temperature), out.data_ptr(), _ptr(lse),
                                       ws.data_ptr(), ws.numel(), _stream()), "decode")
        return out

    def decode_step(self, q: torch.Tensor, k_new: torch.Tensor, v_new: torch.Tensor,
                    temperature: float = 1.0, out: torch.Tensor | None = None,
                    lse: torch.Tensor | None = None) -> torch.Tensor:
        """One generation step (Algorithm 1): append the new token of every unit
        (k_new, v_new [U, d]) at row n, then decode q [U, G, d] over rows [0, n + 1).
        On the tcgen05 path the append is fused into the step's query-sketch kernel;
        otherwise it runs as K1 + value quantizer launches before the decode."""
        if temperature <= 0:
            raise ValueError(f"temperature must be positive, got {temperature}")
        s = self.shape
        q = self._check_q(q)
        kn, vn = k_new.contiguous(), v_new.contiguous()
        if tuple(kn.shape) != (s.units, s.d) or tuple(vn.shape) != (s.units, s.d):
            raise ValueError(f"new token must be [units, d] = [{s.units}, {s.d}]")
        if self.n != self.n_values:
            raise ValueError(f"cache holds {self.n} keys but {self.n_values} value tokens")
        if self.n + 1 > s.capacity:
            raise ValueError(f"cache capacity {s.capacity} exceeded")
        G = q.shape[1]
        if out is None:
            out = torch.empty(s.units, G, s.d, dtype=torch.float32, device=self.device)
        kd, vd, sd = self.key_desc(), self.value_desc(), self.sketch_desc()
        n = self.n
        ws_b = int(self.lib.qjl_decode_workspace(ctypes.byref(kd), ctypes.byref(vd), n + 1, G))
        ws = self.workspace(ws_b)
        rc = -2
        if kn.dtype == q.dtype and vn.dtype == q.dtype:
            rc = self.lib.qjl_decode_step(ctypes.byref(kd), ctypes.byref(vd), n, q.data_ptr(),
                                          _TORCH2QJL[q.dtype], G, ctypes.byref(sd), self.channels.data_ptr(),
                                          s.h, kn.data_ptr(), vn.data_ptr(), 1.0 / float(temperature),
                                          out.data_ptr(), _ptr(lse), ws.data_ptr(), ws.numel(), _stream())
        if rc == _lib.QJL_ERR_UNSUPPORTED:
            self.append(kn[:, None, :], vn[:, None, :])
            return self.decode(q, temperature, out=out, lse=lse)
        _lib.check(rc, "decode_step")
        self.n += 1
        self.n_values += 1
        return out

    # ------------------------------------------------------------- factory    # ------------------------------------------------------------- factory
    @classmethod
    def create(cls, units: int, d: int, m_in: int, h: int = 0, m_out: int | None = None,
               capacity: int = 4096, seed: int = 0, orthogonalize_sketches: bool = True,
               channels=None, key_dtype: torch.dtype = torch.bfloat16, **kw) -> "DeviceKeyCache":
        """Mirror of KeyCacheState.create (kvcache.py:234-267) for U units sharing one
        seed: S_in = G(m_in, d-h, derive_seed(seed, 0)), S_out = G(m_out, h,
        derive_seed(seed, 1)), m_out defaulting to 8*h."""
        if m_out is None:
            m_out = DEFAULT_OUTLIER_BITS_PER_CHANNEL * h
        m_in_eff = m_in if d - h > 0 else 0
        c = cls(units, d, m_in_eff, m_out if h else 0, h, capacity, key_dtype=key_dtype, **kw)
        if channels is not None:
            c.set_channels(channels)
        S_in, S_out = cls.make_sketches(d, h, m_in_eff, m_out if h else 0, seed,
                                        orthogonalize_sketches, _TORCH2NAME[c.sketch_dtype])
        c.seed, c.orthogonalized = seed, orthogonalize_sketches
        c.S_in_host, c.S_out_host = S_in, S_out
        if channels is not None or h == 0:
            c.set_sketches(S_in, S_out)
        return c

    # ------------------------------------------------------------- host views
    def host_view(self, n: int | None = None) -> dict:
        """Copy the packed cache to host numpy (for tests / QJLC export)."""
        n = self.n if n is None else n
        r = dict(bits_in=self.bits_in[:, :n].cpu().numpy(),
                 norm_in=self.norm_in[:, :n].float().cpu().numpy().astype(np.float64))
        if self.bits_out is not None:
            r["bits_out"] = self.bits_out[:, :n].cpu().numpy()
            r["norm_out"] = self.norm_out[:, :n].float().cpu().numpy().astype(np.float64)
        return r


def _p2_tables():
    """Byte offset (within a 4 KB tile) and bit shift of every (token, dim) of a
    128-token P2 tile -- the host mirror of `p2_pos` in csrc/common.cuh."""
    t = np.arange(128)[:, None]
    d = np.arange(128)[None, :]
    sl, j, i = (t >> 5) & 3, t & 7, (t >> 3) & 3
    mt, g, r = d >> 4, d & 7, (d >> 3) & 1
    k, s = mt >> 1, 2 * (mt & 1) + r
    word = sl * 256 + (g * 8 + (j ^ ((g & 1) << 2))) * 4 + k
    byte = word * 4 + i
    return (np.broadcast_to(byte, (128, 128)).astype(np.int64),
            np.broadcast_to(2 * s, (128, 128)).astype(np.uint8))


_P2_BYTE, _P2_SHIFT = _p2_tables()


def _p2t_tables():
    """P2T byte offset / shift of every (token, dim) of a 128-token tile (`p2t_pos`)."""
    t = np.arange(128)[:, None]
    d = np.arange(128)[None, :]
    byte = (d >> 2) * 128 + (t >> 2) * 4 + (t & 3)
    return (np.broadcast_to(byte, (128, 128)).astype(np.int64),
            np.broadcast_to(2 * (d & 3), (128, 128)).astype(np.uint8))


_P2T_BYTE, _P2T_SHIFT = _p2t_tables()


def unpack_codes(packed: np.ndarray, n: int | None = None, layout: str = "p2") -> np.ndarray:
    """Host decoder of a packed 2-bit code layout ("p2" or "p2t") -> codes [..., n, 128]."""
    return p2_unpack_codes(packed, n, layout)


def p2_unpack_codes(packed: np.ndarray, n: int | None = None, layout: str = "p2") -> np.ndarray:
    """Host decoder of the P2 tile-interleaved code layout: packed u8 [..., cap, 32]
    (cap a multiple of 128, rows counted from the unit's row 0) -> codes [..., n, 128]."""
    packed = np.ascontiguousarray(packed, dtype=np.uint8)
    cap = packed.shape[-2]
    if cap % 128:
        raise ValueError("P2 code arrays hold whole 128-token tiles")
    tiles = packed.reshape(packed.shape[:-2] + (cap // 128, 4096))
    bt, sh = (_P2T_BYTE, _P2T_SHIFT) if layout == "p2t" else (_P2_BYTE, _P2_SHIFT)
    codes = (tiles[..., bt] >> sh) & 3
    codes = codes.reshape(packed.shape[:-2] + (cap, 128)).astype(np.uint8)
    return codes if n is None else codes[..., :n, :]


def p2_pack_codes(codes: np.ndarray, layout: str = "p2") -> np.ndarray:
    """Inverse of p2_unpack_codes: codes [..., n, 128] -> packed u8 [..., cap, 32],
    cap = n rounded up to whole 128-token tiles (padding codes are 0)."""
    codes = np.asarray(codes, np.uint8)
    n = codes.shape[-2]
    cap = (n + 127) // 128 * 128
    full = np.zeros(codes.shape[:-2] + (cap, 128), np.uint8)
    full[..., :n, :] = codes & 3
    tiles = full.reshape(codes.shape[:-2] + (cap // 128, 128 * 128))
    out = np.zeros(codes.shape[:-2] + (cap // 128, 4096), np.uint8)
    bt, sh = (_P2T_BYTE, _P2T_SHIFT) if layout == "p2t" else (_P2_BYTE, _P2_SHIFT)
    flat_byte = bt.reshape(-1)
    flat_shift = sh.reshape(-1)
    order = np.argsort(flat_byte, kind="stable")          # 4 (token, dim) per byte
    contrib = (tiles[..., order].astype(np.uint32) << flat_shift[order]).reshape(
        codes.shape[:-2] + (cap // 128, 4096, 4)).sum(-1)
    out[...] = contrib.astype(np.uint8)
    return out.reshape(codes.shape[:-2] + (cap, 32))
