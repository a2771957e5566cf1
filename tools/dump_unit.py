"""Dump one unit's logits / value cache (and both decode outputs) for offline emulation."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2406_03482_b200.device import p2_unpack_codes
from tests.test_decode_tc_gpu import _both, _cache
U, n, G = 64, 4096, 4
c, q = _cache(U, n, G, 8, 256, 64, seed=U * 7 + n)
T = float(np.sqrt(128))
a, b = _both(c, q, T)
lg = c.scores(q).double().cpu().numpy()
np.savez_compressed("gpurun_out/unit0.npz", logits=lg[0], codes=p2_unpack_codes(c.v_codes[0].cpu().numpy(), n, c.value_layout),
                    zero=c.v_zero[0, :n].double().cpu().numpy(), scale=c.v_scale[0, :n].double().cpu().numpy(),
                    out_tc=a[0], out_simt=b[0], T=T)
print("dumped")
