"""GPU parity: the CUDA path (through the C ABI) against the pinned CPU oracle
on identical seeded inputs, at sizes the oracle finishes in seconds.
Shapes follow BASELINE.json configs 1-4 (reduced n / units)."""

import zlib

import numpy as np
import pytest
import torch

from oracle import qjl_oracle as O
from tests._parity import (OUT_RTOL, check_logits, flip_report, logit_bound, make_inputs,
                           rel_l2)

pytestmark = pytest.mark.gpu

TD = {"f32": torch.float32, "f16": torch.float16, "bf16": torch.bfloat16}
NPD = {"f32": np.float32, "f16": np.float16, "bf16": None}


def _round_keys(x, dt):
    t = torch.from_numpy(x).to(TD[dt])
    return t, t.double().numpy()


def _build(cuda, units, n, d, G, h, factor, m_in, m_out, dt, seed, orth=True, layout="p2t",
           device_profile=True, lognormal=False):
    from paper_2406_03482_b200.device import DeviceKeyCache

    K, V, Q, planted = make_inputs(units, n, d, G, h, factor, seed, lognormal)
    Kt, Kr = _round_keys(K, dt)
    Vt, Vr = _round_keys(V, dt)
    Qt, Qr = _round_keys(Q, dt)
    cache = DeviceKeyCache.create(units, d, m_in, h=h, m_out=m_out, capacity=n + 64, seed=seed,
                                  orthogonalize_sketches=orth, key_dtype=TD[dt],
                                  value_layout=layout,
                                  value_group=32 if layout == "p2t" else d)
    if h:
        if device_profile:
            ch = cache.detect_outliers(Kt.to(cuda)).cpu().numpy()
        else:
            cache.set_channels(planted)
            ch = np.array(planted)
        cache.set_sketches(cache.S_in_host, cache.S_out_host)
        chans = [tuple(int(c) for c in row) for row in ch]
    else:
        chans = [()] * units
    cache.append(Kt.to(cuda), Vt.to(cuda))
    torch.cuda.synchronize()
    return cache, Kr, Vr, Qt, Qr, chans, planted


@pytest.mark.parametrize("dt", ["f32", "bf16"])
def test_c1_quantize_and_scores(cuda, dt):
    """Config 1: 1x8 heads, n=1024, m=256, h=0, i.i.d. S, fp32 keys (plus bf16)."""
    U, n, d, m = 8, 1024, 128, 256
    cache, Kr, _, Qt, Qr, _, _ = _build(cuda, U, n, d, 1, 0, 1.0, m, 0, dt, seed=1, orth=False)
    hv = cache.host_view()
    S = cache.S_in_host
    tot = dict(total=0, lt1e6=0, coords=0)
    for u in range(U):
        r = O.append_keys(S, None, (), Kr[u])
        fr = flip_report(hv["bits_in"][u], r["bits_in"], r["proj_in"], m)
        tot["total"] += fr["total"]; tot["lt1e6"] += fr["lt1e6"]; tot["coords"] += fr["coords"]
        assert np.array_equal(hv["norm_in"][u], O.fp16_round(r["norm_in"]))
    print("flip report", tot)
    assert tot["total"] == tot["lt1e6"], tot
    logits = cache.scores(Qt.to(cuda)).cpu().numpy()
    for u in range(U):
        c = dict(bits_in=hv["bits_in"][u], norm_in=hv["norm_in"][u])
        ref = O.estimate_logits(S, None, (), Qr[u, 0], c)
        ok, err = check_logits(logits[u, 0].astype(np.float64), ref,
                               logit_bound(S, None, (), Qr[u, 0], hv["norm_in"][u], 0))
        assert ok.all(), (u, err.max())


@pytest.mark.parametrize("cfg", [
    # name, U, n, G, h, factor, m_in, m_out, dtype, values-layout
    ("c2", 4, 1024, 1, 4, 15.0, 256, 128, "f16", "p2t"),
    ("c3", 4, 2048, 4, 8, 20.0, 256, 64, "bf16", "p2t"),
    ("c3_odd_n", 2, 1000, 4, 8, 20.0, 256, 64, "bf16", "p2t"),
    ("m512", 2, 777, 2, 8, 20.0, 512, 64, "bf16", "p2t"),
    ("u8_ref_values", 2, 700, 2, 4, 15.0, 256, 128, "f16", "u8"),
])
def test_decode_parity(cuda, cfg):
    name, U, n, G, h, factor, m_in, m_out, dt, layout = cfg
    d = 128
    cache, Kr, Vr, Qt, Qr, chans, planted = _build(cuda, U, n, d, G, h, factor, m_in, m_out, dt,
                                                   seed=zlib.crc32(name.encode()) % 1000, layout=layout)
    # outlier profile: device == oracle (fp64 both sides)
    for u in range(U):
        assert chans[u] == O.detect_outliers(Kr[u], h)[0] == planted[u]
    hv = cache.host_view()
    S_in, S_out = cache.S_in_host, cache.S_out_host
    flips = 0
    caches = []
    for u in range(U):
        r = O.append_keys(S_in, S_out, chans[u], Kr[u])
        fi = flip_report(hv["bits_in"][u], r["bits_in"], r["proj_in"], m_in)
        fo = flip_report(hv["bits_out"][u], r["bits_out"], r["proj_out"], m_out)
        assert fi["total"] == fi["lt1e6"] and fo["total"] == fo["lt1e6"], (fi, fo)
        flips += fi["total"] + fo["total"]
        assert np.array_equal(hv["norm_in"][u], O.fp16_round(r["norm_in"]))
        assert np.array_equal(hv["norm_out"][u], O.fp16_round(r["norm_out"]))
        caches.append(dict(bits_in=hv["bits_in"][u], bits_out=hv["bits_out"][u],
                           norm_in=hv["norm_in"][u], norm_out=hv["norm_out"][u]))
    # value codes/constants == oracle quantizer (fp64 both sides, fp16 constants)
    group = 32 if layout == "p2t" else d
    deq = np.zeros_like(Vr)
    for u in range(U):
        codes, zero, scale = O.quantize_values(Vr[u], 2, group,
                                               const_dtype="f16" if layout == "p2t" else None)
        if layout == "p2t":
            from paper_2406_03482_b200.device import unpack_codes
            dc = unpack_codes(cache.v_codes[u].cpu().numpy(), n)
            assert np.array_equal(dc, codes)
            assert np.array_equal(cache.v_zero[u, :n].double().cpu().numpy(), zero)
            assert np.array_equal(cache.v_scale[u, :n].double().cpu().numpy(), scale)
        else:
            assert np.array_equal(cache.v_codes[u, :n].cpu().numpy(), codes)
            zero = cache.v_zero[u, :n].double().cpu().numpy()   # f32 storage of the constants
            scale = cache.v_scale[u, :n].double().cpu().numpy()
        deq[u] = O.dequantize_values(codes, zero, scale)
    for T in (1.0, float(np.sqrt(d))):
        out = cache.decode(Qt.to(cuda), temperature=T).cpu().numpy()
        ref, ref_logits = O.decode_units(S_in, S_out, chans, Qr, caches, deq, T)
        for u in range(U):
            for g in range(G):
                e = rel_l2(out[u, g].astype(np.float64), ref[u, g])
                assert e <= OUT_RTOL, (name, T, u, g, e)
    logits = cache.scores(Qt.to(cuda)).cpu().numpy()
    for u in range(U):
        for g in range(G):
            ok, err = check_logits(logits[u, g].astype(np.float64), ref_logits[u, g],
                                   logit_bound(S_in, S_out, chans[u], Qr[u, g],
                                               caches[u]["norm_in"], caches[u]["norm_out"]))
            assert ok.all(), (name, u, g, err.max())


def test_prefill_c4_shape_small(cuda):
    """Config 4 envelope: m=512, r=8, bf16 keys with lognormal channel scales."""
    cache, Kr, _, _, _, chans, _ = _build(cuda, 4, 1024, 128, 1, 8, 1.0, 512, 64, "bf16", seed=44,
                                          lognormal=True)
    hv = cache.host_view()
    for u in range(4):
        r = O.append_keys(cache.S_in_host, cache.S_out_host, chans[u], Kr[u])
        fi = flip_report(hv["bits_in"][u], r["bits_in"], r["proj_in"], 512)
        fo = flip_report(hv["bits_out"][u], r["bits_out"], r["proj_out"], 64)
        assert fi["total"] == fi["lt1e6"] and fo["total"] == fo["lt1e6"], (fi, fo)


def test_edge_cases(cuda):
    from paper_2406_03482_b200.device import DeviceKeyCache

    d = 128
    c = DeviceKeyCache.create(2, d, 256, h=0, capacity=64, seed=3, key_dtype=torch.float32)
    q = torch.randn(2, 1, d, device=cuda)
    with pytest.raises(ValueError):
        c.scores(q)                       # empty cache (kvcache.py:324-325)
    with pytest.raises(ValueError):
        c.decode(q)
    k = torch.zeros(2, 1, d, device=cuda)                       # zero key
    v = torch.full((2, 1, d), 5.0, device=cuda)                 # constant value token
    c.append(k, v)
    assert torch.all(c.bits_in[:, 0] == 0xFF) and torch.all(c.norm_in[:, 0] == 0)
    assert torch.all(c.v_scale[:, 0] == 0) and torch.all(c.v_codes[:, 0] == 0)
    lg = c.scores(q)
    assert torch.all(lg == 0)                                   # nu = 0 -> exactly 0
    out = c.decode(q)                                           # n = 1 -> weight 1
    torch.testing.assert_close(out, torch.full_like(out, 5.0), rtol=0, atol=0)
    with pytest.raises(ValueError):
        c.decode(q, temperature=0.0)
    with pytest.raises(ValueError):
        c.append_keys(torch.zeros(2, 1, 64, device=cuda))       # dim mismatch


def test_prefix_invariance_bitwise(cuda):
    """Append-only: logits/outputs of the first n0 tokens do not change after
    more appends -- bitwise on the device."""
    from paper_2406_03482_b200.device import DeviceKeyCache

    torch.manual_seed(0)
    U, d = 4, 128
    c = DeviceKeyCache.create(U, d, 256, h=0, capacity=4096, seed=9)
    K = torch.randn(U, 3000, d, device=cuda, dtype=torch.bfloat16)
    V = torch.randn(U, 3000, d, device=cuda, dtype=torch.bfloat16)
    q = torch.randn(U, 4, d, device=cuda, dtype=torch.bfloat16)
    c.append(K[:, :2000], V[:, :2000])
    l1 = c.scores(q).clone()
    o1 = c.decode(q, deterministic=True).clone()
    c.append(K[:, 2000:], V[:, 2000:])
    l2 = c.scores(q, n=2000)
    o2 = c.decode(q, n=2000, deterministic=True)
    assert torch.equal(l1, l2[..., :2000])
    assert torch.equal(o1, o2)
    # chunked appends == one-shot append (partition independence)
    c2 = DeviceKeyCache.create(U, d, 256, h=0, capacity=4096, seed=9)
    c2.append(K, V)
    assert torch.equal(c2.bits_in[:, :3000], c.bits_in[:, :3000])
    assert torch.equal(c2.v_codes[:, :3000], c.v_codes[:, :3000])
