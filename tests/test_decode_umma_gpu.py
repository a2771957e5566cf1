"""tcgen05 fused decode (k_decode_umma.cu, P2T value caches) checks: against the generic
SIMT path on the same device cache, across stream-K unit boundaries and tail tiles, at
the full config-3 size against the CPU oracle on sampled units, and the P2T code
layout round trip through the device value quantizer."""

import numpy as np
import pytest
import torch

from oracle import qjl_oracle as O
from tests._parity import OUT_RTOL, rel_l2
from tests.test_decode_tc_gpu import _both, _cache

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("U,n,G,h,m_in,m_out", [
    (64, 4096, 4, 8, 256, 64),      # many CTAs per unit, segments cross units
    (8, 100, 4, 8, 256, 64),        # fewer tiles than CTAs, tail tile
    (3, 1, 2, 8, 256, 64),          # n = 1
    (16, 2000, 1, 4, 256, 128),     # MHA, config-2 sketch sizes
    (4, 3000, 4, 0, 256, 0),        # no outliers
    (4, 3000, 3, 8, 512, 64),       # m = 512, G = 3
    (8, 5000, 2, 8, 256, 64),       # G = 2 (two-head epilogue)
    (6, 2500, 1, 8, 512, 64),       # G = 1 with m = 512 (one-head epilogue)
])
def test_umma_matches_simt(cuda, U, n, G, h, m_in, m_out):
    c, q = _cache(U, n, G, h, m_in, m_out, seed=U * 7 + n, layout="p2t")
    for T in (1.0, float(np.sqrt(128))):
        a, b = _both(c, q, T)
        for u in range(U):
            for g in range(G):
                assert rel_l2(a[u, g], b[u, g]) <= 1e-4, (u, g, T, rel_l2(a[u, g], b[u, g]))


def test_umma_full_config3_against_oracle(cuda):
    from paper_2406_03482_b200.device import p2_unpack_codes

    U, n, G = 64, 32768, 4
    c, q = _cache(U, n, G, 8, 256, 64, seed=3, layout="p2t")
    out = c.decode(q).double().cpu().numpy()
    Qh = q.double().cpu().numpy()
    assert np.isfinite(out).all()
    for u in (0, U - 1):
        chans = tuple(int(x) for x in c.channels[u, :8].cpu().numpy())
        cache = dict(bits_in=c.bits_in[u, :n].cpu().numpy(),
                     norm_in=c.norm_in[u, :n].double().cpu().numpy(),
                     bits_out=c.bits_out[u, :n].cpu().numpy(),
                     norm_out=c.norm_out[u, :n].double().cpu().numpy())
        codes = p2_unpack_codes(c.v_codes[u].cpu().numpy(), n, "p2t")
        deq = O.dequantize_values(codes, c.v_zero[u, :n].double().cpu().numpy(),
                                  c.v_scale[u, :n].double().cpu().numpy())
        for g in range(G):
            ref, _, _ = O.quantized_decode(c.S_in_host, c.S_out_host, chans, Qh[u, g], cache, deq)
            assert rel_l2(out[u, g], ref) <= OUT_RTOL, (u, g, rel_l2(out[u, g], ref))


def test_p2t_codes_match_oracle_quantizer(cuda):
    from paper_2406_03482_b200.device import DeviceKeyCache, p2_unpack_codes

    U, n = 3, 300
    V = torch.randn(U, n, 128, device="cuda", dtype=torch.bfloat16)
    c = DeviceKeyCache(U, 128, 256, 0, 0, n, value_layout="p2t")
    c.append_values(V)
    Vh = V.double().cpu().numpy()
    for u in range(U):
        codes, zero, scale = O.quantize_values(Vh[u], 2, 32)
        assert np.array_equal(p2_unpack_codes(c.v_codes[u].cpu().numpy(), n, "p2t"), codes)


def test_umma_lse_and_determinism(cuda):
    c, q = _cache(8, 5000, 4, 8, 256, 64, seed=11, layout="p2t")
    lse1 = torch.empty(8, 4, device="cuda")
    o1 = c.decode(q, lse=lse1).clone()
    o2 = c.decode(q)
    assert torch.equal(o1, o2)
    lg = c.scores(q).double()
    ref_lse = torch.logsumexp(lg, dim=-1)
    torch.testing.assert_close(lse1.double(), ref_lse, rtol=1e-4, atol=1e-3)


def test_p2t_quantizer_exact_ties_and_unaligned_appends(cuda):
    """Values on a grid that puts many quotients exactly on .5 (round-half-even in the
    reference), constant groups, and appends starting at rows that are not multiples of 4."""
    from paper_2406_03482_b200.device import DeviceKeyCache, p2_unpack_codes

    U, n = 2, 203
    g = torch.Generator().manual_seed(5)
    V = (torch.randint(0, 7, (U, n, 128), generator=g).double() * 0.5)   # multiples of 1/2 -> ties
    V[:, 7, 32:64] = 1.25                                                   # constant group
    V[:, 11] *= 1e-3
    Vt = V.to(torch.bfloat16)
    c = DeviceKeyCache(U, 128, 256, 0, 0, n, value_layout="p2t")
    for a, b in ((0, 5), (5, 6), (6, 70), (70, 203)):                       # unaligned row offsets
        c.append_values(Vt[:, a:b].to(cuda))
    Vh = Vt.double().numpy()
    for u in range(U):
        codes, zero, scale = O.quantize_values(Vh[u], 2, 32, const_dtype="f16")
        assert np.array_equal(p2_unpack_codes(c.v_codes[u].cpu().numpy(), n, "p2t"), codes)
        assert np.array_equal(c.v_zero[u, :n].double().cpu().numpy(), zero)
        assert np.array_equal(c.v_scale[u, :n].double().cpu().numpy(), scale)


def test_warp_specialized_kernel_matches(cuda):
    """The opt-in warp-specialized variant (QJL_UD_WS=1) against the default kernel."""
    import os

    c, q = _cache(64, 4096, 4, 8, 256, 64, seed=21, layout="p2t")
    a = c.decode(q).double().cpu().numpy()
    os.environ["QJL_UD_WS"] = "1"
    try:
        b = c.decode(q).double().cpu().numpy()
    finally:
        del os.environ["QJL_UD_WS"]
    from tests._parity import rel_l2
    for u in range(64):
        for g in range(4):
            assert rel_l2(b[u, g], a[u, g]) <= 1e-4, (u, g)
