"""Tensor-core fused decode (k_decode_tc.cu) checks: against the generic SIMT
path on the same device cache (QJL_FORCE_SIMT selects it), across stream-K
unit boundaries and tail tiles, and at the full config-3 size against the CPU
oracle on sampled units."""

import os

import numpy as np
import pytest
import torch

from oracle import qjl_oracle as O
from tests._parity import OUT_RTOL, rel_l2

pytestmark = pytest.mark.gpu


def _cache(U, n, G, h, m_in, m_out, seed, dtype=torch.bfloat16, factor=20.0, layout="p2"):
    from paper_2406_03482_b200.device import DeviceKeyCache

    gen = torch.Generator(device="cuda")
    gen.manual_seed(seed)
    K = torch.randn(U, n, 128, generator=gen, device="cuda")
    if h:
        ch = torch.argsort(torch.rand(U, 128, generator=gen, device="cuda"), dim=1)[:, :h]
        sc = torch.ones(U, 128, device="cuda").scatter_(1, ch, factor)
        K = K * sc[:, None, :]
    V = torch.randn(U, n, 128, generator=gen, device="cuda")
    Qx = torch.randn(U, G, 128, generator=gen, device="cuda")
    K, V, Qx = K.to(dtype), V.to(dtype), Qx.to(dtype)
    c = DeviceKeyCache.create(U, 128, m_in, h=h, m_out=m_out, capacity=n, seed=seed, key_dtype=dtype,
                              value_layout=layout)
    if h:
        c.detect_outliers(K)
        c.set_sketches(c.S_in_host, c.S_out_host)
    c.append(K, V)
    return c, Qx


def _both(c, q, T=1.0):
    os.environ["QJL_REQUIRE_TC"] = "1"          # no silent fallback to the generic kernel
    try:
        out_tc = c.decode(q, temperature=T).clone()
    finally:
        del os.environ["QJL_REQUIRE_TC"]
    os.environ["QJL_FORCE_SIMT"] = "1"
    try:
        out_simt = c.decode(q, temperature=T).clone()
    finally:
        del os.environ["QJL_FORCE_SIMT"]
    return out_tc.double().cpu().numpy(), out_simt.double().cpu().numpy()


@pytest.mark.parametrize("U,n,G,h,m_in,m_out", [
    (64, 4096, 4, 8, 256, 64),      # many CTAs per unit, segments cross units
    (8, 100, 4, 8, 256, 64),        # fewer tiles than CTAs, tail tile
    (3, 1, 2, 8, 256, 64),          # n = 1
    (16, 2000, 1, 4, 256, 128),     # MHA, config-2 sketch sizes
    (4, 3000, 4, 0, 256, 0),        # no outliers
    (4, 3000, 3, 8, 512, 64),       # m = 512, G = 3
])
def test_tc_matches_simt(cuda, U, n, G, h, m_in, m_out):
    c, q = _cache(U, n, G, h, m_in, m_out, seed=U * 7 + n)
    for T in (1.0, float(np.sqrt(128))):
        a, b = _both(c, q, T)
        for u in range(U):
            for g in range(G):
                assert rel_l2(a[u, g], b[u, g]) <= 2e-4, (u, g, T, rel_l2(a[u, g], b[u, g]))


def test_tc_full_config3_against_oracle(cuda):
    """Full config-3 shape (64 units x 32768 tokens, 4 q-heads/unit) through the
    fast path; the oracle checks 2 sampled units (first and last)."""
    from paper_2406_03482_b200.device import p2_unpack_codes

    U, n, G = 64, 32768, 4
    c, q = _cache(U, n, G, 8, 256, 64, seed=3)
    out = c.decode(q).double().cpu().numpy()
    Qh = q.double().cpu().numpy()
    assert np.isfinite(out).all()
    for u in (0, U - 1):
        chans = tuple(int(x) for x in c.channels[u, :8].cpu().numpy())
        cache = dict(bits_in=c.bits_in[u, :n].cpu().numpy(),
                     norm_in=c.norm_in[u, :n].double().cpu().numpy(),
                     bits_out=c.bits_out[u, :n].cpu().numpy(),
                     norm_out=c.norm_out[u, :n].double().cpu().numpy())
        codes = p2_unpack_codes(c.v_codes[u].cpu().numpy(), n)
        deq = O.dequantize_values(codes, c.v_zero[u, :n].double().cpu().numpy(),
                                  c.v_scale[u, :n].double().cpu().numpy())
        for g in range(G):
            ref, _, _ = O.quantized_decode(c.S_in_host, c.S_out_host, chans, Qh[u, g], cache, deq)
            assert rel_l2(out[u, g], ref) <= OUT_RTOL, (u, g, rel_l2(out[u, g], ref))


def test_tc_lse_and_determinism(cuda):
    c, q = _cache(8, 5000, 4, 8, 256, 64, seed=11)
    lse1 = torch.empty(8, 4, device="cuda")
    o1 = c.decode(q, lse=lse1).clone()
    o2 = c.decode(q)
    assert torch.equal(o1, o2)                      # deterministic (no atomics)
    lg = c.scores(q).double()                        # generic logits
    ref_lse = torch.logsumexp(lg, dim=-1)
    torch.testing.assert_close(lse1.double(), ref_lse, rtol=1e-4, atol=1e-3)
