"""Device caches with seeded torch inputs, and the oracle's view of them (the same packed
sign bits, fp16 norms and fp16 value constants the device holds -- SURVEY 8(c) steps 5-6).
Used by the tensor-core decode / scores tests."""

from __future__ import annotations

import numpy as np
import torch

from oracle import qjl_oracle as O


def make_cache(U, n, G, h, m_in, m_out, seed, dtype=torch.bfloat16, factor=20.0, capacity=None):
    """A tile-major P2T cache with n tokens of seeded N(0,1) keys (h planted outlier
    channels x factor), values and G query heads per unit."""
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
    c = DeviceKeyCache.create(U, 128, m_in, h=h, m_out=m_out, capacity=capacity or n, seed=seed,
                              key_dtype=dtype)
    if h:
        c.detect_outliers(K)
        c.set_sketches(c.S_in_host, c.S_out_host)
    c.append(K, V)
    return c, Qx


def oracle_unit(c, u, n=None):
    """(channels, packed key cache dict, dequantized values) of unit u as the oracle sees them."""
    from paper_2406_03482_b200.device import unpack_codes

    n = c.n if n is None else n
    s = c.shape
    chans = tuple(int(x) for x in c.channels[u, :s.h].cpu().numpy()) if s.h else ()
    cache = dict(bits_in=c.bits_in[u, :n].cpu().numpy(), norm_in=c.norm_in[u, :n].double().cpu().numpy())
    if s.m_out:
        cache["bits_out"] = c.bits_out[u, :n].cpu().numpy()
        cache["norm_out"] = c.norm_out[u, :n].double().cpu().numpy()
    codes = unpack_codes(c.v_codes[u].cpu().numpy(), n)
    deq = O.dequantize_values(codes, c.v_zero[u, :n].double().cpu().numpy(),
                              c.v_scale[u, :n].double().cpu().numpy())
    return chans, cache, deq


def oracle_decode(c, q, u, T=1.0, n=None):
    """Oracle outputs [G, d], weights and logits [G, n] (natural-log units, before 1/T)."""
    chans, cache, deq = oracle_unit(c, u, n)
    Qh = q[u].double().cpu().numpy()
    outs, logits = [], []
    for g in range(Qh.shape[0]):
        out, _, lg = O.quantized_decode(c.S_in_host, c.S_out_host, chans, Qh[g], cache, deq, T)
        outs.append(out)
        logits.append(lg)
    return np.stack(outs), np.stack(logits)


def logsumexp(x):
    m = x.max(axis=-1, keepdims=True)
    return (m + np.log(np.exp(x - m).sum(axis=-1, keepdims=True)))[..., 0]
