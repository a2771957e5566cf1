"""Shared parity helpers: seeded inputs, oracle evaluation with the device's
storage policy (fp16 norms / constants, operand-rounded S), tolerance checks
from BASELINE.json's north star:

  * sign bits: bit-exact except projections with |(Sk)_j| < 1e-6 (flips counted)
  * logits:   |d| <= 1e-3 |ref|  or  |d| <= 1e-6 * sqrt(pi/2)/m * nu * ||Sq||_1 (per side)
  * outputs:  relative L2 <= 1e-3 (fp32 accumulation)
"""

from __future__ import annotations

import numpy as np

from oracle import qjl_oracle as O
from paper_2406_03482_b200.sketch import derive_seed, rng_from_seed

BIT_EPS = 1e-6
LOGIT_RTOL = 1e-3
LOGIT_COND = 1e-6
OUT_RTOL = 1e-3


def make_inputs(units, n, d, G, h, factor, seed, lognormal=False):
    """Seeded synthetic K, V, Q (harness.py:38-42 stream ids) with `h` planted
    outlier channels per unit scaled by `factor`."""
    rk = rng_from_seed(derive_seed(seed, 0))
    rv = rng_from_seed(derive_seed(seed, 1))
    rq = rng_from_seed(derive_seed(seed, 2))
    rc = rng_from_seed(derive_seed(seed, 3))
    K = rk.standard_normal((units, n, d))
    planted = []
    for u in range(units):
        ch = np.sort(rc.choice(d, size=h, replace=False)) if h else np.zeros(0, int)
        K[u][:, ch] *= factor
        planted.append(tuple(int(c) for c in ch))
        if lognormal:
            K[u] *= np.exp(rc.standard_normal(d))[None, :]
    V = rv.standard_normal((units, n, d))
    Q = rq.standard_normal((units, G, d))
    return K, V, Q, planted


def flip_report(dev_bits, ref_bits, proj, m):
    """Count mismatching sign bits, bucketed by |projection|."""
    db = O.unpack_rows(dev_bits, m)
    rb = O.unpack_rows(ref_bits, m)
    bad = db != rb
    a = np.abs(proj)[bad]
    return dict(total=int(bad.sum()), lt1e6=int((a < 1e-6).sum()),
                lt1e5=int(((a >= 1e-6) & (a < 1e-5)).sum()),
                lt1e4=int(((a >= 1e-5) & (a < 1e-4)).sum()), ge1e4=int((a >= 1e-4).sum()),
                coords=int(bad.size))


def logit_bound(S_in, S_out, channels, q, norm_in, norm_out):
    """Condition-aware absolute bound per token."""
    inl, outl = O.split_index(q.shape[0], channels)
    b = LOGIT_COND * O.ESTIMATOR_SCALE / S_in.shape[0] * norm_in * np.abs(S_in @ q[inl]).sum()
    if len(outl):
        b = b + LOGIT_COND * O.ESTIMATOR_SCALE / S_out.shape[0] * norm_out * np.abs(S_out @ q[outl]).sum()
    return b


def check_logits(dev, ref, bound):
    err = np.abs(dev - ref)
    ok = (err <= LOGIT_RTOL * np.abs(ref)) | (err <= bound)
    return ok, err


def rel_l2(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))
