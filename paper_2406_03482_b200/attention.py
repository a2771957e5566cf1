"""Drop-in mirror of `pkg/src/qjl/attention.py::quantized_decode` on the device.

`quantized_decode(query, state, value_tokens, temperature)` (attention.py:56-71)
runs the fused decode kernel (scores -> softmax -> weights @ dequantized values)
over the state's device key cache and a value cache built from the reference
value tokens (U8 layout: 1 byte per code, per-token zero/scale), and returns the
same DecodeResult(output float64 [d], scores ScoreVector).  `exact_decode` and
the error metrics are the reference's full-precision comparison tools, not part
of the quantized path, and are out of scope here.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .device import _stream
from .kvcache import KeyCacheState, QuantizedValueToken, ScoreVector, _softmax_rows


@dataclass(frozen=True, eq=False)
class DecodeResult:
    """Attention output vector and the scores that produced it (attention.py:25-30)."""

    output: np.ndarray
    scores: ScoreVector


def quantized_decode(query: np.ndarray, state: KeyCacheState, value_tokens: list[QuantizedValueToken],
                     temperature: float = 1.0) -> DecodeResult:
    """Attention decode from a quantized cache on the B200 (attention.py:56-71)."""
    if state.n == 0:
        raise ValueError("cache is empty")
    if len(value_tokens) != state.n:
        raise ValueError(f"cache holds {state.n} keys but {len(value_tokens)} value tokens supplied")
    if temperature <= 0:
        raise ValueError(f"temperature must be positive, got {temperature}")
    bits = value_tokens[0].bits
    d = state.d
    if any(t.bits != bits or t.d != d for t in value_tokens):
        raise ValueError("value tokens must share one bit width and dimension")
    lib = _lib.load()
    n = state.n
    dev = state.device_cache.device
    codes = torch.from_numpy(np.stack([t.codes for t in value_tokens]).astype(np.uint8)).to(dev)[None]
    zero = torch.tensor([[float(t.zero)] for t in value_tokens], dtype=torch.float32, device=dev)[None]
    scale = torch.tensor([[float(t.scale)] for t in value_tokens], dtype=torch.float32, device=dev)[None]
    vd = _lib.ValueCacheDesc(codes.data_ptr(), zero.data_ptr(), scale.data_ptr(), n, 1, d, bits, d,
                             _lib.QJL_VLAYOUT_U8, 0, 0)
    c = state.device_cache
    c.n = n
    kd, sd = c.key_desc(), c.sketch_desc()
    q = state._query_tensor(query)
    out = torch.empty(1, 1, d, dtype=torch.float32, device=dev)
    logits = torch.empty(1, n, dtype=torch.float32, device=dev)    # logits / T of this launch
    ws_b = int(lib.qjl_decode_workspace(ctypes.byref(kd), ctypes.byref(vd), n, 1))
    ws = c.workspace(ws_b)
    _lib.check(lib.qjl_decode(ctypes.byref(kd), ctypes.byref(vd), n, q.data_ptr(), _lib.QJL_F64, 1,
                              ctypes.byref(sd), 1.0 / float(temperature), out.data_ptr(), None,
                              logits.data_ptr(), ws.data_ptr(), ws.numel(), 0, _stream()), "quantized_decode")
    # the ScoreVector is the fp64 softmax of the logits the fused decode itself consumed
    weights = _softmax_rows(logits, 1.0)[0]
    return DecodeResult(output=out[0, 0].double().cpu().numpy(), scores=ScoreVector(weights=weights))
