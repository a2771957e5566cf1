"""Decode-step append (the paper's Algorithm 1): qjl_decode_step
quantizes each unit's new token inside the step's query-sketch kernel and decodes over
the grown cache.  Checked against the separate K1 + value-quantizer appends followed by
the decode (bit for bit: same cache bytes, same outputs) and against the CPU oracle."""

import numpy as np
import pytest
import torch

from oracle import qjl_oracle as O
from paper_2406_03482_b200.device import DeviceKeyCache, unpack_codes
from tests._parity import rel_l2

pytestmark = pytest.mark.gpu


def _pair(U, n0, G, h, m_in, m_out, seed, layout="p2t", cap=None):
    gen = torch.Generator(device="cuda").manual_seed(seed)
    K = torch.randn(U, n0 + 8, 128, generator=gen, device="cuda")
    if h:
        ch = torch.argsort(torch.rand(U, 128, generator=gen, device="cuda"), dim=1)[:, :h]
        K = K * torch.ones(U, 128, device="cuda").scatter_(1, ch, 20.0)[:, None, :]
    V = torch.randn(U, n0 + 8, 128, generator=gen, device="cuda")
    Q = torch.randn(U, 8, G, 128, generator=gen, device="cuda")
    K, V, Q = K.bfloat16(), V.bfloat16(), Q.bfloat16()
    caches = []
    for _ in range(2):
        c = DeviceKeyCache.create(U, 128, m_in, h=h, m_out=m_out, capacity=cap or (n0 + 8), seed=seed,
                                  value_layout=layout)
        if h:
            c.detect_outliers(K[:, : max(n0, 1)])
            c.set_sketches(c.S_in_host, c.S_out_host)
        if n0:
            c.append(K[:, :n0], V[:, :n0])
        caches.append(c)
    return caches, K, V, Q


def _arrays(c, n):
    r = [c.bits_in[:, :n], c.norm_in[:, :n], c.v_zero[:, :n], c.v_scale[:, :n]]
    if c.bits_out is not None:
        r += [c.bits_out[:, :n], c.norm_out[:, :n]]
    return r


@pytest.mark.parametrize("U,n0,G,h,m_in,m_out", [
    (64, 1000, 4, 8, 256, 64),      # C3 sketch sizes
    (16, 127, 1, 4, 256, 128),      # MHA, the new token opens a tile
    (8, 0, 2, 8, 256, 64),          # first token of an empty cache
    (4, 300, 3, 0, 256, 0),         # no outliers
])
def test_decode_step_equals_append_then_decode(cuda, U, n0, G, h, m_in, m_out):
    (a, b), K, V, Q = _pair(U, n0, G, h, m_in, m_out, seed=n0 + U)
    for i in range(5):                                    # five consecutive generation steps
        t = n0 + i
        out_a = a.decode_step(Q[:, i], K[:, t], V[:, t], deterministic=True).clone()
        b.append(K[:, t:t + 1], V[:, t:t + 1])
        out_b = b.decode(Q[:, i], deterministic=True)
        assert a.n == b.n == t + 1
        for x, y in zip(_arrays(a, t + 1), _arrays(b, t + 1)):
            assert torch.equal(x, y)
        ca = unpack_codes(a.v_codes.cpu().numpy(), t + 1)
        cb = unpack_codes(b.v_codes.cpu().numpy(), t + 1)
        assert np.array_equal(ca, cb)
        assert torch.equal(out_a, out_b)


def test_decode_step_against_oracle(cuda):
    U, n0, G = 4, 700, 4
    (a, _), K, V, Q = _pair(U, n0, G, 8, 256, 64, seed=5)
    out = a.decode_step(Q[:, 0], K[:, n0], V[:, n0]).double().cpu().numpy()
    n = n0 + 1
    S_in, S_out = a.S_in_host, a.S_out_host
    Kh, Vh, Qh = K.double().cpu().numpy(), V.double().cpu().numpy(), Q[:, 0].double().cpu().numpy()
    for u in range(U):
        ch = tuple(int(x) for x in a.channels[u].cpu())
        cache = O.append_keys(S_in, S_out, ch, Kh[u, :n])
        cache["norm_in"], cache["norm_out"] = O.fp16_round(cache["norm_in"]), O.fp16_round(cache["norm_out"])
        codes, zero, scale = O.quantize_values(Vh[u, :n], 2, 32)
        deq = O.dequantize_values(codes, zero, scale)
        for g in range(G):
            ref, _, _ = O.quantized_decode(S_in, S_out, ch, Qh[u, g], cache, deq)
            assert rel_l2(out[u, g], ref) <= 1e-3


def test_decode_step_chained_and_u8_fallback(cuda):
    """Chained steps (QJL_DECODE_CHAINED) equal unchained ones; u8 caches (the generic
    decode) run append + decode."""
    (a, b), K, V, Q = _pair(4, 200, 4, 8, 256, 64, seed=9)
    for i in range(4):
        oa = a.decode_step(Q[:, i], K[:, 200 + i], V[:, 200 + i], chained=i > 0, deterministic=True).clone()
        ob = b.decode_step(Q[:, i], K[:, 200 + i], V[:, 200 + i], deterministic=True)
        assert torch.equal(oa, ob)
    c = DeviceKeyCache.create(4, 128, 256, h=0, capacity=300, value_layout="u8", value_group=128)
    c.append(K[:, :200], V[:, :200])
    out = c.decode_step(Q[:, 0], K[:, 200], V[:, 200])
    assert c.n == c.n_values == 201 and torch.isfinite(out).all()
    with pytest.raises(ValueError):
        c = DeviceKeyCache.create(2, 128, 256, h=0, capacity=128)
        c.append(torch.randn(2, 128, 128, device="cuda").bfloat16(), torch.randn(2, 128, 128, device="cuda").bfloat16())
        c.decode_step(torch.randn(2, 4, 128, device="cuda").bfloat16(), torch.randn(2, 128, device="cuda").bfloat16(),
                      torch.randn(2, 128, device="cuda").bfloat16())   # capacity exceeded
