"""Diagnose TC vs SIMT vs oracle on one failing configuration."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from oracle import qjl_oracle as O
from tests.test_decode_tc_gpu import _cache, _both
from paper_2406_03482_b200.device import p2_unpack_codes
U, n, G = 64, 4096, 4
c, q = _cache(U, n, G, 8, 256, 64, seed=U * 7 + n)
T = float(np.sqrt(128))
a, b = _both(c, q, T)
Qh = q.double().cpu().numpy()
for u in (2, 5):
    chans = tuple(int(x) for x in c.channels[u, :8].cpu().numpy())
    cache = dict(bits_in=c.bits_in[u, :n].cpu().numpy(), norm_in=c.norm_in[u, :n].double().cpu().numpy(),
                 bits_out=c.bits_out[u, :n].cpu().numpy(), norm_out=c.norm_out[u, :n].double().cpu().numpy())
    codes = p2_unpack_codes(c.v_codes[u].cpu().numpy(), n)
    z = c.v_zero[u, :n].double().cpu().numpy(); s = c.v_scale[u, :n].double().cpu().numpy()
    deq = O.dequantize_values(codes, z, s)
    for g in range(G):
        ref, w, lg = O.quantized_decode(c.S_in_host, c.S_out_host, chans, Qh[u, g], cache, deq, T)
        et = a[u, g] - ref; es = b[u, g] - ref
        print(f"u{u} g{g} |ref|={np.linalg.norm(ref):.3f} maxw={w.max():.3f} "
              f"tc rel={np.linalg.norm(et)/np.linalg.norm(ref):.2e} simt rel={np.linalg.norm(es)/np.linalg.norm(ref):.2e}")
        print("   tc err per group:", [f"{np.abs(et[k*32:(k+1)*32]).mean():.1e}" for k in range(4)],
              " simt:", [f"{np.abs(es[k*32:(k+1)*32]).mean():.1e}" for k in range(4)])
        # component split: zero term and code term
        zt = (w[:, None] * np.repeat(z, 32, axis=1)).sum(0)
        ct = (w[:, None] * codes * np.repeat(s, 32, axis=1)).sum(0)
        print("   |zero term| per group:", [f"{np.abs(zt[k*32]):.2f}" for k in range(4)],
              " |code term|:", [f"{np.abs(ct[k*32:(k+1)*32]).mean():.2f}" for k in range(4)])
