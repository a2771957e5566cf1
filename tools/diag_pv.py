"""Separate the zero-point and code terms of the TC PV path against the SIMT path."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from tests.test_decode_tc_gpu import _cache, _both
T = float(np.sqrt(128))
for n in (512, 4096, 32768):
    c, q = _cache(16, n, 4, 8, 256, 64, seed=7)
    def err(tag):
        a, b = _both(c, q, T)
        e = np.abs(a - b).max(axis=-1) / np.abs(b).max(axis=-1)
        off = (a - b).mean(axis=-1) / np.abs(b).mean(axis=-1)
        print(f"n={n:6d} {tag:12s} max rel {e.max():.2e}  mean signed offset {off.mean():+.2e}")
    err("full")
    z0, s0 = c.v_zero.clone(), c.v_scale.clone()
    c.v_scale.zero_(); err("zero only")
    c.v_scale.copy_(s0); c.v_zero.zero_(); err("codes only")
    c.v_zero.fill_(1.0); c.v_scale.zero_(); err("zero=1")
    c.v_zero.zero_(); c.v_scale.fill_(1.0); c.v_codes.fill_(0x55); err("codes=1")
