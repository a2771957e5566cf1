"""Isolate TC logit precision: with n = 1 the decode lse equals the token's scaled logit."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from tests.test_decode_tc_gpu import _cache
for (h, mo) in ((8, 64), (0, 0)):
    U, G = 512, 4
    c, q = _cache(U, 1, G, h, 256, mo, seed=5)
    lse = torch.empty(U, G, device="cuda")
    c.decode(q, lse=lse)
    lg = c.scores(q)[..., 0]
    d = (lse - lg).abs()
    rel = d / lg.abs().clamp_min(1e-3)
    print(f"h={h}: |logit| median {lg.abs().median().item():.3f}  abs err max {d.max().item():.3e} "
          f"median {d.median().item():.3e}  rel max {rel.max().item():.3e} median {rel.median().item():.3e}")
    i = int(d.flatten().argmax())
    print("   worst", lg.flatten()[i].item(), lse.flatten()[i].item())
