"""tcgen05 + TMA key quantizer (k_quant_tc.cu) checks: bit-identical to the fp64
generic path on the same inputs (QJL_REQUIRE_TC forbids a silent fallback),
tails / chunked appends at row offsets, and the full config-4 size against the
CPU oracle on sampled units."""

import os

import numpy as np
import pytest
import torch

from oracle import qjl_oracle as O
from tests._parity import flip_report

pytestmark = pytest.mark.gpu


def _keys(U, n, dt, seed, lognormal=True, h=0, factor=20.0):
    g = torch.Generator(device="cuda")
    g.manual_seed(seed)
    K = torch.randn(U, n, 128, generator=g, device="cuda")
    if lognormal:
        K = K * torch.exp(torch.randn(U, 1, 128, generator=g, device="cuda"))
    if h:
        ch = torch.argsort(torch.rand(U, 128, generator=g, device="cuda"), dim=1)[:, :h]
        K = K * torch.ones(U, 128, device="cuda").scatter_(1, ch, factor)[:, None, :]
    return K.to(dt)


def _quantize(K, m_in, h, m_out, dt, path, chunks=1):
    from paper_2406_03482_b200.device import DeviceKeyCache

    U, n, _ = K.shape
    c = DeviceKeyCache.create(U, 128, m_in, h=h, m_out=m_out, capacity=n, seed=3, key_dtype=dt,
                              with_values=False)
    if h:
        c.detect_outliers(K)
        c.set_sketches(c.S_in_host, c.S_out_host)
    env = {"tc": ("QJL_REQUIRE_TC", "1"), "simt": ("QJL_FORCE_SIMT", "1")}[path]
    os.environ[env[0]] = env[1]
    try:
        bounds = np.linspace(0, n, chunks + 1).astype(int)
        for a, b in zip(bounds[:-1], bounds[1:]):
            c.append_keys(K[:, a:b].contiguous())
    finally:
        del os.environ[env[0]]
    torch.cuda.synchronize()
    return c


@pytest.mark.parametrize("U,n,m_in,h,m_out,dt", [
    (2, 300, 256, 0, 0, torch.bfloat16),      # config-1 sketch, tail tile
    (4, 1000, 256, 8, 64, torch.bfloat16),    # configs 3/5
    (3, 700, 256, 4, 128, torch.float16),     # config 2 (fp16)
    (4, 2048, 512, 8, 64, torch.bfloat16),    # config 4
    (2, 129, 512, 0, 0, torch.float16),       # m = 512, one full + one 1-row tile
])
def test_tc_bitwise_equals_fp64_path(cuda, U, n, m_in, h, m_out, dt):
    K = _keys(U, n, dt, seed=U * 1000 + n, h=h)
    a = _quantize(K, m_in, h, m_out, dt, "tc")
    b = _quantize(K, m_in, h, m_out, dt, "simt")
    assert torch.equal(a.bits_in[:, :n], b.bits_in[:, :n])
    assert torch.equal(a.norm_in[:, :n], b.norm_in[:, :n])
    if m_out:
        assert torch.equal(a.bits_out[:, :n], b.bits_out[:, :n])
        assert torch.equal(a.norm_out[:, :n], b.norm_out[:, :n])


def test_tc_chunked_appends_equal_one_shot(cuda):
    """Append-only semantics: appending in 3 chunks at row offsets == one append."""
    K = _keys(4, 1500, torch.bfloat16, seed=7, h=8)
    a = _quantize(K, 256, 8, 64, torch.bfloat16, "tc", chunks=1)
    b = _quantize(K, 256, 8, 64, torch.bfloat16, "tc", chunks=3)
    assert torch.equal(a.bits_in[:, :1500], b.bits_in[:, :1500])
    assert torch.equal(a.bits_out[:, :1500], b.bits_out[:, :1500])
    assert torch.equal(a.norm_in[:, :1500], b.norm_in[:, :1500])


def test_tc_config4_full_size_against_oracle(cuda):
    """Config 4: B16 x Hkv8 = 128 units x 8192 keys, m = 512 + 64, r = 8, lognormal
    channel scales; 2 sampled units through the oracle (bits exact except |Sk| < 1e-6)."""
    U, n = 128, 8192
    K = _keys(U, n, torch.bfloat16, seed=44)
    c = _quantize(K, 512, 8, 64, torch.bfloat16, "tc")
    for u in (0, U - 1):
        Kr = K[u].double().cpu().numpy()
        chans = tuple(int(x) for x in c.channels[u, :8].cpu().numpy())
        assert chans == O.detect_outliers(Kr, 8)[0]
        r = O.append_keys(c.S_in_host, c.S_out_host, chans, Kr)
        fi = flip_report(c.bits_in[u, :n].cpu().numpy(), r["bits_in"], r["proj_in"], 512)
        fo = flip_report(c.bits_out[u, :n].cpu().numpy(), r["bits_out"], r["proj_out"], 64)
        assert fi["total"] == fi["lt1e6"] and fo["total"] == fo["lt1e6"], (fi, fo)
        assert np.array_equal(c.norm_in[u, :n].double().cpu().numpy(), O.fp16_round(r["norm_in"]))
        assert np.array_equal(c.norm_out[u, :n].double().cpu().numpy(), O.fp16_round(r["norm_out"]))
