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
    """Packed QJL key cache + 2-bit (or u8) value cache for `units` units.

    Layouts (include/qjl_b200.h):
      * "p2t" values (the tensor-core path): tile-major records -- one contiguous
        record per (unit, 128-token tile) holding sign bits, fp16 norms, 2-bit codes and
        fp16 zero/scale (`qjl_tile_record`), so the decode streams one bulk copy per tile;
      * "u8" values (the reference's own format): separate row-major arrays;
      * keys only (`with_values=False`): tile-major records of the key fields when
        `tiled` (the tensor-core scores kernel), else row-major arrays.
    The per-field properties (`bits_in`, `norm_in`, ..., `v_codes`) are dense
    [units, capacity, ...] tensors: views in the rows layout, COPIES (read-only) in the
    tile-major one; write into a tiled cache only through the library or `field_view`.
    """

    def __init__(self, units: int, d: int, m_in: int, m_out: int, h: int, capacity: int, *,
                 key_dtype: torch.dtype = torch.bfloat16, value_bits: int = 2,
                 value_group: int = 32, value_layout: str = "p2t", with_values: bool = True,
                 sketch_dtype: torch.dtype | None = None, device: str | torch.device = "cuda",
                 validate_rate: bool = True, tiled: bool | None = None):
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
        if with_values and value_layout not in ("p2t", "u8"):
            raise ValueError(f"unknown value layout {value_layout!r}")
        self.device = torch.device(device)
        # rows are padded to whole 128-token tiles: the tensor-core decode streams
        # full tiles with bulk copies and masks tokens >= n
        capacity = (capacity + 127) // 128 * 128
        self.shape = CacheShape(units, d, m_in, m_out, h, capacity)
        self.key_dtype = key_dtype
        self.sketch_dtype = sketch_dtype or operand_dtype_for(key_dtype)
        self.value_layout = value_layout
        self.with_values = with_values
        self.value_bits, self.value_group = value_bits, value_group
        p2t = with_values and value_layout == "p2t"
        if p2t and not (d == 128 and value_bits == 2 and value_group == 32):
            raise ValueError("p2t value layout is 2-bit, group 32, d = 128")
        if tiled is None:
            tiled = p2t or (not with_values and m_in % 32 == 0 and m_out % 32 == 0)
        if p2t and not tiled:
            raise ValueError("p2t values live in tile-major records")
        if with_values and not p2t and tiled:
            raise ValueError("u8 values use the rows layout")
        self.tiled = tiled
        dev = self.device
        self.channels = torch.zeros(units, max(h, 1), dtype=torch.int32, device=dev)
        self.s_full: torch.Tensor | None = None
        self.n = 0
        self.n_values = 0
        self._ws: torch.Tensor | None = None
        Gv = d // value_group
        if tiled:
            offs = (ctypes.c_int64 * 7)()
            rec = int(self.lib.qjl_tile_record(d, m_in, m_out, 1 if p2t else 0, offs))
            if rec <= 0:
                raise ValueError(f"no tile record for d={d}, m_in={m_in}, m_out={m_out}")
            self.record_bytes = rec
            self.record_offsets = list(offs)
            tiles = capacity // 128
            self._bind_records(torch.zeros(units, tiles, rec, dtype=torch.uint8, device=dev))
        else:
            self.record_bytes = 0
            self._fields = None
            self._bits_in = torch.zeros(units, capacity, max(m_in, 8) // 8, dtype=torch.uint8, device=dev)
            self._norm_in = torch.zeros(units, capacity, dtype=torch.float16, device=dev)
            self._bits_out = (torch.zeros(units, capacity, m_out // 8, dtype=torch.uint8, device=dev)
                              if m_out else None)
            self._norm_out = torch.zeros(units, capacity, dtype=torch.float16, device=dev) if m_out else None
            if with_values:
                self._v_codes = torch.zeros(units, capacity, d, dtype=torch.uint8, device=dev)
                self._v_zero = torch.zeros(units, capacity, Gv, dtype=torch.float32, device=dev)
                self._v_scale = torch.zeros(units, capacity, Gv, dtype=torch.float32, device=dev)

    # ------------------------------------------------------------ fields
    def _bind_records(self, records: torch.Tensor) -> None:
        """Point the cache at a [units, tiles, record_bytes] record buffer and build the
        per-field views into it (offsets from qjl_tile_record)."""
        s = self.shape
        units, tiles = s.units, s.capacity // 128
        Gv = s.d // self.value_group
        self.records = records
        self._fields = {}

        def fld(i, width, dtype=torch.uint8):
            o = self.record_offsets[i]
            v = records[:, :, o:o + 128 * width * (torch.finfo(dtype).bits // 8
                                                    if dtype.is_floating_point else 1)]
            v = v.view(dtype) if dtype != torch.uint8 else v
            return v.view(units, tiles, 128, width)

        self._fields["bits_in"] = fld(_lib.QJL_REC_BITS_IN, s.m_in // 8)
        self._fields["norm_in"] = fld(_lib.QJL_REC_NORM_IN, 1, torch.float16)
        if s.m_out:
            self._fields["bits_out"] = fld(_lib.QJL_REC_BITS_OUT, s.m_out // 8)
            self._fields["norm_out"] = fld(_lib.QJL_REC_NORM_OUT, 1, torch.float16)
        if self.value_layout == "p2t" and self.with_values:
            self._fields["v_codes"] = fld(_lib.QJL_REC_CODES, s.d // 4)
            self._fields["v_zero"] = fld(_lib.QJL_REC_ZERO, Gv, torch.float16)
            self._fields["v_scale"] = fld(_lib.QJL_REC_SCALE, Gv, torch.float16)

    def replica(self) -> "DeviceKeyCache":
        """A second cache with the same contents in its own record buffer (same sketches,
        channels and workspace).  bench.py rotates decodes over replicas so that a shard
        smaller than L2 is still read from HBM."""
        if not self.tiled:
            raise ValueError("replica() is for tile-major caches")
        import copy

        r = copy.copy(self)
        r._bind_records(self.records.clone())
        return r

    def field_view(self, name: str) -> torch.Tensor:
        """Writable view of one cache field: [units, tiles, 128, width] (tile-major) or
        the dense [units, capacity, ...] array (rows layout)."""
        if self.tiled:
            if name not in self._fields:
                raise KeyError(name)
            return self._fields[name]
        t = getattr(self, "_" + name, None)
        if t is None:
            raise KeyError(name)
        return t

    def _dense(self, name: str):
        if not self.tiled:
            return getattr(self, "_" + name, None)
        v = self._fields.get(name)
        if v is None:
            return None
        s = self.shape
        out = v.reshape(s.units, s.capacity, v.shape[-1])
        return out[..., 0] if name in ("norm_in", "norm_out") else out

    bits_in = property(lambda self: self._dense("bits_in"))
    bits_out = property(lambda self: self._dense("bits_out"))
    norm_in = property(lambda self: self._dense("norm_in"))
    norm_out = property(lambda self: self._dense("norm_out"))
    v_codes = property(lambda self: self._dense("v_codes"))
    v_zero = property(lambda self: self._dense("v_zero"))
    v_scale = property(lambda self: self._dense("v_scale"))

    def fill_rows(self, name: str, rows: slice, value: float) -> None:
        """Set a field of rows `rows` of every unit to `value` (both layouts)."""
        t = self.field_view(name)
        if not self.tiled:
            t[:, rows] = value
            return
        idx = torch.arange(self.shape.capacity, device=self.device)[rows]
        t[:, idx // 128, idx % 128] = value

    def tensor_core_path(self, G: int, scores: bool = False) -> bool:
        """True when decode (or scores) with G query heads runs the tensor-core kernels."""
        kd = self.key_desc()
        if scores or not self.with_values:
            return self.lib.qjl_tensor_core_path(ctypes.byref(kd), None, G) == 1
        vd = self.value_desc()
        return self.lib.qjl_tensor_core_path(ctypes.byref(kd), ctypes.byref(vd), G) == 1

    # ------------------------------------------------------------ descriptors
    def _ptr_of(self, name: str) -> int | None:
        if self.tiled:
            v = self._fields.get(name)
            return None if v is None else v.data_ptr()
        t = getattr(self, "_" + name, None)
        return None if t is None else t.data_ptr()

    def key_desc(self) -> _lib.KeyCacheDesc:
        s = self.shape
        return _lib.KeyCacheDesc(self._ptr_of("bits_in"), self._ptr_of("bits_out"), self._ptr_of("norm_in"),
                                 self._ptr_of("norm_out"), s.capacity, s.units, s.d, s.m_in, s.m_out,
                                 self.record_bytes)

    def value_desc(self) -> _lib.ValueCacheDesc:
        s = self.shape
        layout = _lib.QJL_VLAYOUT_P2T if self.value_layout == "p2t" else _lib.QJL_VLAYOUT_U8
        return _lib.ValueCacheDesc(self._ptr_of("v_codes"), self._ptr_of("v_zero"), self._ptr_of("v_scale"),
                                   s.capacity, s.units, s.d, self.value_bits, self.value_group,
                                   layout, 0, self.record_bytes)

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

    def _detect_ws(self, n0: int) -> torch.Tensor:
        """The outlier detection's partials buffer (qjl_detect_workspace), kept across calls."""
        nb = int(self.lib.qjl_detect_workspace(self.shape.units, n0, self.shape.d))
        if getattr(self, "_dws", None) is None or self._dws.numel() < nb:
            self._dws = torch.empty(max(nb, 1), dtype=torch.uint8, device=self.device)
        return self._dws

    def workspace(self, nbytes: int) -> torch.Tensor:
        if self._ws is None or self._ws.numel() < nbytes:
            # zero-filled: the tensor-core decode keeps its merge counters at the start
            self._ws = torch.zeros(max(nbytes, 1), dtype=torch.uint8, device=self.device)
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
        ws = self._detect_ws(pk.shape[1])
        _lib.check(self.lib.qjl_detect_outliers(pk.data_ptr(), _TORCH2QJL[pk.dtype], s.units,
                                                pk.shape[1], s.d, pk.shape[1] * s.d, s.h,
                                                self.channels.data_ptr(), mags.data_ptr(),
                                                ws.data_ptr(), ws.numel(), _stream()), "detect_outliers")
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
        """Prompt profile + append: `qjl_prefill_profile` detects each unit's
        outlier channels and builds its zero-padded S_full in one pass over the prompt
        (kvcache.py:104-123, :234-267), then K1 quantizes the prompt into rows [n, n + n0)
        (kvcache.py:293-306) and the values, if given, are quantized alongside."""
        self.prefill_profile(prompt_keys)
        self.append(prompt_keys.contiguous(), values)

    def prefill_profile(self, prompt_keys: torch.Tensor) -> None:
        """The profile alone (`qjl_prefill_profile`): channels, magnitudes and S_full from the
        prompt, no quantization (kvcache.py:104-123, :234-267)."""
        s = self.shape
        pk = prompt_keys.contiguous()
        if pk.dim() != 3 or pk.shape[0] != s.units or pk.shape[2] != s.d or pk.shape[1] == 0:
            raise ValueError("prompt keys must be a non-empty [units, n0, d] tensor")
        if getattr(self, "S_in_host", None) is None and getattr(self, "S_out_host", None) is None:
            raise ValueError("no host sketches: build the cache with DeviceKeyCache.create")
        dev = self.device
        if getattr(self, "_sk_op", None) is None:
            self._sk_op = tuple(None if S is None else
                                torch.as_tensor(np.ascontiguousarray(S, np.float64)).to(dev, self.sketch_dtype)
                                for S in (self.S_in_host, self.S_out_host))
        sin, sout = self._sk_op
        if self.s_full is None:
            self.s_full = torch.empty(s.units, s.m_in + s.m_out, s.d, dtype=self.sketch_dtype, device=dev)
        mags = torch.empty(s.units, s.d, dtype=torch.float64, device=dev)
        ws = self._detect_ws(pk.shape[1])
        _lib.check(self.lib.qjl_prefill_profile(pk.data_ptr(), _TORCH2QJL[pk.dtype], s.units, pk.shape[1],
                                                s.d, pk.shape[1] * s.d, s.h, _ptr(sin), _ptr(sout),
                                                s.m_in, s.m_out, _TORCH2QJL[self.sketch_dtype],
                                                self.channels.data_ptr(), mags.data_ptr(),
                                                self.s_full.data_ptr(), ws.data_ptr(), ws.numel(),
                                                _stream()), "prefill_profile")
        self.magnitudes = mags

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
                                             s.d, ctypes.byref(sd), s.m_in + s.m_out, _lib.QJL_F32,
                                             out.data_ptr(), _stream()), "sketch_query")
        return out

    def scores(self, q: torch.Tensor, n: int | None = None, out: torch.Tensor | None = None,
               chained: bool = False) -> torch.Tensor:
        """K2: logits [U, G, n] f32 (kvcache.py:311-329).  `chained`: as for `decode`
        (QJL_DECODE_CHAINED) -- the previous kernel on the stream is this library's scores or
        decode and every input predates it."""
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
                                       _lib.QJL_DECODE_CHAINED if chained else 0, _stream()), "scores")
        return out

    def decode_workspace_bytes(self, G: int, n: int | None = None) -> int:
        n = self.n if n is None else n
        kd, vd = self.key_desc(), self.value_desc()
        return int(self.lib.qjl_decode_workspace(ctypes.byref(kd), ctypes.byref(vd), n, G))

    def decode(self, q: torch.Tensor, temperature: float = 1.0, n: int | None = None,
               out: torch.Tensor | None = None, lse: torch.Tensor | None = None,
               chained: bool = False, logits: torch.Tensor | None = None,
               deterministic: bool = False) -> torch.Tensor:
        """K2+K3: softmax(logits / T) @ V per query head -> [U, G, d] f32 (attention.py:56-71).
        `chained`: the previous kernel on the stream is this cache's decode and every input
        predates it (QJL_DECODE_CHAINED) -- lets the query sketch overlap that decode.
        `deterministic`: fixed per-unit segments (QJL_DECODE_DETERMINISTIC), so each unit's
        output is independent of the other units in the call (sharding-invariant bits)."""
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
                                       1.0 / float(temperature), out.data_ptr(), _ptr(lse), _ptr(logits),
                                       ws.data_ptr(), ws.numel(),
                                       (_lib.QJL_DECODE_CHAINED if chained else 0) |
                                       (_lib.QJL_DECODE_DETERMINISTIC if deterministic else 0), _stream()), "decode")
        return out

    def bench_decode_kernel(self, q: torch.Tensor, reps: int, temperature: float = 1.0,
                            out: torch.Tensor | None = None, deterministic: bool = False) -> float:
        """Mean time (ms) of the tensor-core decode kernel in a chain of `reps` back-to-back
        decodes (qjl_bench_decode_kernel): the roofline kernel as it runs in a decode loop."""
        s = self.shape
        q = self._check_q(q)
        G = q.shape[1]
        if out is None:
            out = torch.empty(s.units, G, s.d, dtype=torch.float32, device=self.device)
        kd, vd, sd = self.key_desc(), self.value_desc(), self.sketch_desc()
        ws_b = int(self.lib.qjl_decode_workspace(ctypes.byref(kd), ctypes.byref(vd), self.n, G))
        ws = self.workspace(ws_b)
        ms = ctypes.c_float(0.0)
        _lib.check(self.lib.qjl_bench_decode_kernel(ctypes.byref(kd), ctypes.byref(vd), self.n, q.data_ptr(),
                                                    _TORCH2QJL[q.dtype], G, ctypes.byref(sd),
                                                    1.0 / float(temperature), out.data_ptr(), None,
                                                    ws.data_ptr(), ws.numel(),
                                                    _lib.QJL_DECODE_DETERMINISTIC if deterministic else 0,
                                                    int(reps), ctypes.byref(ms), _stream()), "bench_decode_kernel")
        return float(ms.value)

    def decode_step(self, q: torch.Tensor, k_new: torch.Tensor, v_new: torch.Tensor,
                    temperature: float = 1.0, out: torch.Tensor | None = None,
                    lse: torch.Tensor | None = None, chained: bool = False,
                    deterministic: bool = False) -> torch.Tensor:
        """One generation step (Algorithm 1): append the new token of every unit
        (k_new, v_new [U, d]) at row n, then decode q [U, G, d] over rows [0, n + 1).
        On the tcgen05 path the append is fused into the step's query-sketch kernel;
        otherwise it runs as K1 + value quantizer launches before the decode.
        `deterministic` selects the fixed-segment schedule (bitwise reproducible)."""
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
                                          out.data_ptr(), _ptr(lse), None, ws.data_ptr(), ws.numel(),
                                          (_lib.QJL_DECODE_CHAINED if chained else 0)
                                          | (_lib.QJL_DECODE_DETERMINISTIC if deterministic else 0), _stream())
        if rc == _lib.QJL_ERR_UNSUPPORTED:
            self.append(kn[:, None, :], vn[:, None, :])
            return self.decode(q, temperature, out=out, lse=lse, deterministic=deterministic)
        _lib.check(rc, "decode_step")
        self.n += 1
        self.n_values += 1
        return out

    # ------------------------------------------------------------- factory
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


def _p2t_tables():
    """P2T byte offset / shift of every (token, dim) of a 128-token tile (`p2t_byte` in
    csrc/common.cuh: dim quad dq = d // 4 owns 128 bytes, its 16-token chunk j stored at
    chunk position j ^ (dq % 4))."""
    t = np.arange(128)[:, None]
    d = np.arange(128)[None, :]
    dq, tw = d >> 2, t >> 2
    byte = dq * 128 + (((tw >> 2) ^ (dq & 3)) << 4) + ((tw & 3) << 2) + (t & 3)
    return (np.broadcast_to(byte, (128, 128)).astype(np.int64),
            np.broadcast_to(2 * (d & 3), (128, 128)).astype(np.uint8))


_P2T_BYTE, _P2T_SHIFT = _p2t_tables()


def unpack_codes(packed: np.ndarray, n: int | None = None) -> np.ndarray:
    """Host decoder of the P2T tile-interleaved code layout: packed u8 [..., cap, 32]
    (cap a multiple of 128, rows counted from the unit's row 0, i.e. the dense
    `DeviceKeyCache.v_codes`) -> codes [..., n, 128]."""
    packed = np.ascontiguousarray(packed, dtype=np.uint8)
    cap = packed.shape[-2]
    if cap % 128:
        raise ValueError("P2T code arrays hold whole 128-token tiles")
    tiles = packed.reshape(packed.shape[:-2] + (cap // 128, 4096))
    codes = (tiles[..., _P2T_BYTE] >> _P2T_SHIFT) & 3
    codes = codes.reshape(packed.shape[:-2] + (cap, 128)).astype(np.uint8)
    return codes if n is None else codes[..., :n, :]


def pack_codes(codes: np.ndarray) -> np.ndarray:
    """Inverse of unpack_codes: codes [..., n, 128] -> packed u8 [..., cap, 32],
    cap = n rounded up to whole 128-token tiles (padding codes are 0)."""
    codes = np.asarray(codes, np.uint8)
    n = codes.shape[-2]
    cap = (n + 127) // 128 * 128
    full = np.zeros(codes.shape[:-2] + (cap, 128), np.uint8)
    full[..., :n, :] = codes & 3
    tiles = full.reshape(codes.shape[:-2] + (cap // 128, 128 * 128))
    flat_byte = _P2T_BYTE.reshape(-1)
    flat_shift = _P2T_SHIFT.reshape(-1)
    order = np.argsort(flat_byte, kind="stable")          # 4 (token, dim) per byte
    contrib = (tiles[..., order].astype(np.uint32) << flat_shift[order]).reshape(
        codes.shape[:-2] + (cap // 128, 4096, 4)).sum(-1)
    return contrib.astype(np.uint8).reshape(codes.shape[:-2] + (cap, 32))
