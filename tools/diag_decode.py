"""Decode accuracy diagnostic: tensor-core path vs SIMT path vs CPU oracle on a few units."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import qjl_oracle as O
from paper_2406_03482_b200.device import p2_unpack_codes
from tests.test_decode_tc_gpu import _both, _cache


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


U, n, G = int(sys.argv[1]), int(sys.argv[2]), 4
layout = sys.argv[3] if len(sys.argv) > 3 else "p2"
c, q = _cache(U, n, G, 8, 256, 64, seed=U * 7 + n, layout=layout)
Qh = q.double().cpu().numpy()
for T in (1.0, float(np.sqrt(128))):
    a, b = _both(c, q, T)
    for u in (0, 1):
        chans = tuple(int(x) for x in c.channels[u, :8].cpu().numpy())
        cache = dict(bits_in=c.bits_in[u, :n].cpu().numpy(), norm_in=c.norm_in[u, :n].double().cpu().numpy(),
                     bits_out=c.bits_out[u, :n].cpu().numpy(), norm_out=c.norm_out[u, :n].double().cpu().numpy())
        codes = p2_unpack_codes(c.v_codes[u].cpu().numpy(), n, layout)
        deq = O.dequantize_values(codes, c.v_zero[u, :n].double().cpu().numpy(), c.v_scale[u, :n].double().cpu().numpy())
        for g in range(G):
            ref, _, _ = O.quantized_decode(c.S_in_host, c.S_out_host, chans, Qh[u, g], cache, deq, temperature=T)
            print(f"T={T:5.2f} u={u} g={g}  tc-oracle {rel(a[u,g], ref):.2e}  simt-oracle {rel(b[u,g], ref):.2e}  "
                  f"tc-simt {rel(a[u,g], b[u,g]):.2e}  mean(tc-ref) {np.mean(a[u,g]-ref):+.2e} mean(simt-ref) {np.mean(b[u,g]-ref):+.2e}")
