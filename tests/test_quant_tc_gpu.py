"""tcgen05 + TMA key quantizer (k_quant_tc.cu) checks: bit-identical to the fp64
generic kernel on the same inputs, tails / chunked appends at row offsets, and the full
config-4 size against the CPU oracle on sampled units.

Dispatch is by shape (api.cu qjl_quantize_keys): bf16/fp16 keys with a sketch of the same
operand dtype run the tensor-core kernel; an fp64 sketch (here: the same operand-rounded
values held in fp64) runs the fp64 kernel -- which is how the reference comparison is made."""

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
    c = _cache(U, m_in, h, m_out, dt, n, path)
    if h:
        c.detect_outliers(K)
    c.set_sketches(c.S_in_host, c.S_out_host)
    bounds = np.linspace(0, n, chunks + 1).astype(int)
    for a, b in zip(bounds[:-1], bounds[1:]):
        c.append_keys(K[:, a:b].contiguous())
    torch.cuda.synchronize()
    return c


def _cache(U, m_in, h, m_out, dt, n, path, channels=None):
    """path "tc": operand-dtype sketch (tensor-core kernel); "fp64": the same operand-rounded
    sketch values held in fp64 (the fp64 kernel)."""
    from paper_2406_03482_b200.device import DeviceKeyCache

    kw = dict(sketch_dtype=torch.float64) if path == "fp64" else {}
    c = DeviceKeyCache.create(U, 128, m_in, h=h, m_out=m_out, capacity=n, seed=3, key_dtype=dt,
                              with_values=False, channels=channels, **kw)
    op = {torch.bfloat16: "bf16", torch.float16: "f16"}[dt]
    c.S_in_host, c.S_out_host = DeviceKeyCache.make_sketches(128, h, m_in, m_out if h else 0, seed=3, operand=op)
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
    b = _quantize(K, m_in, h, m_out, dt, "fp64")
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


@pytest.mark.parametrize("dt", [torch.bfloat16, torch.float16])
def test_tc_special_rows_match_fp64_path(cuda, dt):
    """Zero / negative-zero / one-side-zero / NaN keys: the tie rule (S k)_i >= 0 -> 1
    (also for -0.0) and NaN -> 0 (estimator.py:119-121) hold on the tensor-core path
    (its accumulators start from +0, so an all-zero dot product is +0)."""
    U, n, h = 2, 256, 8
    K = _keys(U, n, dt, seed=77, h=h)
    ch = torch.stack([torch.randperm(128, generator=torch.Generator().manual_seed(u))[:h].sort().values
                      for u in range(U)]).cuda()
    K[:, 0] = 0.0                                  # all-zero key
    K[:, 1] = -0.0                                 # negative zeros everywhere
    K[:, 2] = K[:, 2].neg()
    for u in range(U):
        K[u, 3, ch[u]] = 0.0                       # outlier side zero, inlier side not
        keep = K[u, 4, ch[u]].clone()
        K[u, 4] = -0.0
        K[u, 4, ch[u]] = keep                      # inlier side (-)zero, outlier side not
    K[:, 5, 7] = float("nan")                      # NaN key

    def run(path):
        c = _cache(U, 256, h, 64, dt, n, path, channels=ch.cpu().numpy())
        c.set_sketches(c.S_in_host, c.S_out_host)
        c.append_keys(K)
        torch.cuda.synchronize()
        return c

    a, b = run("tc"), run("fp64")
    for x, y in ((a.bits_in, b.bits_in), (a.bits_out, b.bits_out)):
        assert torch.equal(x[:, :n], y[:, :n])
    assert torch.all(a.bits_in[:, 0] == 0xFF) and torch.all(a.bits_out[:, 0] == 0xFF)
    assert torch.all(a.bits_in[:, 1] == 0xFF) and torch.all(a.bits_out[:, 1] == 0xFF)
    assert torch.all(a.bits_out[:, 3] == 0xFF) and torch.all(a.bits_in[:, 4] == 0xFF)
    for x, y in ((a.norm_in, b.norm_in), (a.norm_out, b.norm_out)):
        assert torch.equal(x[:, :n].view(torch.int16), y[:, :n].view(torch.int16))
