"""Fused prompt profile: qjl_prefill_profile = detect_outliers +
per-unit S_full build in one pass over the prompt, then K1.  Checked bit for bit against
the separate launches and against the oracle (kvcache.py:104-123, :234-267)."""

import numpy as np
import pytest
import torch

from oracle import qjl_oracle as O
from paper_2406_03482_b200.device import DeviceKeyCache

pytestmark = pytest.mark.gpu


def _keys(U, n0, d, dtype, seed):
    g = torch.Generator(device="cuda").manual_seed(seed)
    k = torch.randn(U, n0, d, device="cuda", generator=g, dtype=torch.float64)
    k = k * torch.exp(torch.randn(U, 1, d, device="cuda", generator=g, dtype=torch.float64))
    return k.to(dtype)


def _pair(U, n0, dtype, h=8, m_in=512, m_out=64, seed=0):
    keys = _keys(U, n0, 128, dtype, seed)
    kw = dict(capacity=n0, seed=seed, key_dtype=dtype, with_values=False)
    a = DeviceKeyCache.create(U, 128, m_in, h=h, m_out=m_out, **kw)
    a.detect_outliers(keys)
    a.set_sketches(a.S_in_host, a.S_out_host)
    a.append_keys(keys)
    b = DeviceKeyCache.create(U, 128, m_in, h=h, m_out=m_out, **kw)
    b.prefill(keys)
    return keys, a, b


@pytest.mark.parametrize("dtype,n0", [(torch.bfloat16, 1000), (torch.float16, 4096), (torch.float32, 777),
                                      (torch.float64, 512), (torch.bfloat16, 300)])
def test_prefill_equals_separate_launches_and_oracle(cuda, dtype, n0):
    U = 5
    keys, a, b = _pair(U, n0, dtype, seed=n0)
    assert torch.equal(a.channels, b.channels)
    assert torch.equal(a.magnitudes, b.magnitudes)
    assert torch.equal(a.s_full, b.s_full)
    for x, y in ((a.bits_in, b.bits_in), (a.bits_out, b.bits_out), (a.norm_in, b.norm_in),
                 (a.norm_out, b.norm_out)):
        assert torch.equal(x[:, :n0], y[:, :n0])
    kh = keys.double().cpu().numpy()
    S_in = a.S_in_host
    S_out = a.S_out_host
    sf = b.s_full.double().cpu().numpy()
    for u in range(U):
        ch, mags = O.detect_outliers(kh[u], 8)
        assert tuple(b.channels[u].cpu().tolist()) == ch
        np.testing.assert_allclose(b.magnitudes[u].cpu().numpy(), mags, rtol=1e-13)
        inl, outl = O.split_index(128, ch)
        want = np.zeros((576, 128))
        want[:512, inl] = S_in
        want[512:, outl] = S_out
        assert np.array_equal(sf[u], want)           # S_in/S_out are already operand-rounded


def test_prefill_without_outliers(cuda):
    keys = _keys(3, 600, 128, torch.bfloat16, 3)
    a = DeviceKeyCache.create(3, 128, 256, h=0, capacity=600, key_dtype=torch.bfloat16, with_values=False)
    a.append_keys(keys)
    b = DeviceKeyCache.create(3, 128, 256, h=0, capacity=600, key_dtype=torch.bfloat16, with_values=False)
    b.prefill(keys)
    assert torch.equal(a.s_full, b.s_full)
    assert torch.equal(a.bits_in[:, :600], b.bits_in[:, :600])


def test_prefill_with_values_and_rate_check(cuda):
    keys = _keys(2, 640, 128, torch.bfloat16, 4)
    vals = _keys(2, 640, 128, torch.bfloat16, 5)
    c = DeviceKeyCache.create(2, 128, 256, h=8, m_out=64, capacity=1024, key_dtype=torch.bfloat16)
    c.prefill(keys, vals)
    assert c.n == 640 and c.n_values == 640
    with pytest.raises(ValueError):           # m_out/h = 8/8 < m_in/(d-h) (kvcache.py:219-226)
        bad = DeviceKeyCache.create(2, 128, 256, h=8, m_out=8, capacity=1024, key_dtype=torch.bfloat16,
                                    validate_rate=False, with_values=False, tiled=False)
        bad.prefill(keys)


def test_prefill_c4_bitwise(cuda):
    """Config 4 (128 units x 8192 keys, m = 512 + 64, r = 8): the fused profile + K1 equals
    detect + build + K1 launched separately, bit for bit -- channels, magnitudes, S_full,
    sign bits and norms."""
    U, n0 = 128, 8192
    keys, a, b = _pair(U, n0, torch.bfloat16, seed=11)
    assert torch.equal(a.channels, b.channels)
    assert torch.equal(a.magnitudes, b.magnitudes)
    assert torch.equal(a.s_full, b.s_full)
    for x, y in ((a.bits_in, b.bits_in), (a.bits_out, b.bits_out), (a.norm_in, b.norm_in),
                 (a.norm_out, b.norm_out)):
        assert torch.equal(x[:, :n0], y[:, :n0])
    # and the profile alone (qjl_prefill_profile) agrees
    c = DeviceKeyCache.create(U, 128, 512, h=8, m_out=64, capacity=n0, seed=11, key_dtype=torch.bfloat16,
                              with_values=False)
    c.prefill_profile(keys)
    assert torch.equal(c.channels, b.channels) and torch.equal(c.magnitudes, b.magnitudes)
    assert torch.equal(c.s_full, b.s_full)


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float16])
def test_detection_exact_with_subnormals_and_zeros(cuda, dtype):
    """The detection kernel adds |x| of 16-bit keys as power-of-two-scaled fp64 values built
    from the magnitude bits (no conversion unit): zeros, subnormals and normals must come
    out as the exact channel means.  Channel groups: subnormals only, subnormals mixed with
    zeros, zeros only, tiny normals, and wide normals -- each group's span keeps its fp64
    sums exact, so the device means equal fsum(|x|) / n bit for bit in any summation order."""
    import math
    U, n0, d = 3, 1000, 128
    g = torch.Generator().manual_seed(5)
    fi = torch.finfo(dtype)
    sub = fi.smallest_normal / (2 ** (7 if dtype == torch.bfloat16 else 10))   # smallest subnormal
    k = torch.empty(U, n0, d, dtype=torch.float64)
    code = torch.randint(1, 128, (U, n0, d), generator=g).double()
    sign = torch.where(torch.rand(U, n0, d, generator=g) < 0.5, -1.0, 1.0).double()
    k[..., 0:32] = code[..., 0:32] * sub                                  # subnormals
    k[..., 32:48] = code[..., 32:48] * sub * (torch.rand(U, n0, 16, generator=g) < 0.5)   # + zeros
    k[..., 48:56] = 0.0
    k[..., 56:80] = torch.rand(U, n0, 24, generator=g).double() * 64 * fi.smallest_normal
    k[..., 80:] = torch.randn(U, n0, d - 80, generator=g).double() * 8
    k = (k * sign).to(dtype)
    c = DeviceKeyCache.create(U, d, 256, h=8, m_out=64, capacity=n0, key_dtype=dtype, with_values=False)
    c.detect_outliers(k.to("cuda"))
    got = c.magnitudes.cpu().numpy()
    kh = k.double().abs().numpy()
    for u in range(U):
        want = np.array([math.fsum(kh[u, :, j]) / n0 for j in range(d)])
        assert np.array_equal(got[u], want), np.flatnonzero(got[u] != want)[:8]
        ch, mags = O.detect_outliers(k[u].double().numpy(), 8)
        assert tuple(c.channels[u].cpu().tolist()) == ch
