"""Statistical suites, host logic: the device harness
(paper_2406_03482_b200/harness.py) with its two device steps replaced by the CPU
oracle reproduces the reports of the real reference harness (tests/golden) --
same seeds, draws, statistics and pass bands."""

import math

import numpy as np
import pytest

from oracle import qjl_oracle as O
from paper_2406_03482_b200 import harness as H
from paper_2406_03482_b200 import sketch as SK

SUITES = {
    "unb_sphere": ("run_unbiasedness_trial", dict(d=64, m=8, trials=300, seed=3, distribution="sphere")),
    "unb_outlier_iid": ("run_unbiasedness_trial", dict(d=32, m=16, trials=200, seed=4, distribution="outlier",
                                                       orthogonalize=False)),
    "dist_m64": ("run_distortion_trial", dict(d=64, m=64, trials=300, seed=5, distribution="gaussian")),
    "dist_m8": ("run_distortion_trial", dict(d=64, m=8, trials=300, seed=5, distribution="gaussian")),
    "scores": ("run_score_trial", dict(d=32, m=64, n=64, trials=100, seed=6)),
    "orth": ("run_orthogonal_comparison", dict(d=64, m=16, trials=300, seed=7)),
}


def _cpu_sketches(m, d, seeds, orthogonalize):
    out = []
    for s in seeds:
        g = SK.generate_gaussian(m, d, int(s))
        out.append((SK.orthogonalize(g) if orthogonalize else g).entries)
    return np.stack(out)


def _cpu_orth(G):
    return np.stack([SK.orthogonalize(SK.SketchMatrix(np.array(g), seed=0)).entries for g in np.asarray(G)])


def _cpu_unit_norm(S, keys, queries):
    T, m, d = S.shape
    out = np.empty((T, keys.shape[1]))
    for t in range(T):
        k = keys[0] if keys.shape[0] == 1 else keys[t]
        bits, _, _ = O.quantize_keys(S[t], k)
        sq = O.sketch_query(S[t], queries[t])
        out[t] = O.ESTIMATOR_SCALE / m * O.packed_sign_dot_batch(bits, m, sq)
    return out


def check_report(row, want, fields, rtol, ztol):
    for f, w in zip(fields, want):
        got = row.get(str(f))
        if np.isnan(w):
            assert got is None, f
        elif f in ("passed", "trials", "failure_fraction", "fraction_within_bound"):
            assert float(got) == w, (f, got, w)
        elif f == "z_score":
            assert abs(got - w) <= ztol, (f, got, w)
        else:
            assert math.isclose(got, w, rel_tol=rtol, abs_tol=1e-12), (f, got, w)


@pytest.mark.parametrize("name", sorted(SUITES))
def test_host_logic_reproduces_reference_reports(golden, monkeypatch, name):
    monkeypatch.setattr(H, "_device_sketches", _cpu_sketches)
    monkeypatch.setattr(H, "orthogonalize_batch", _cpu_orth)
    monkeypatch.setattr(H, "_unit_norm_estimates", _cpu_unit_norm)
    fn, kw = SUITES[name]
    row = getattr(H, fn)(H.TrialConfig(**kw)).to_row()
    check_report(row, golden[f"harness_{name}"], golden["harness_fields"], rtol=1e-9, ztol=1e-7)


def test_config_validation_and_required_m():
    with pytest.raises(ValueError):
        H.TrialConfig(trials=10)
    with pytest.raises(ValueError):
        H.TrialConfig(distribution="cauchy")
    with pytest.raises(ValueError):
        H.TrialConfig(epsilon=1.5)
    assert H.required_m(0.25, 0.01) == 142
    assert H.required_m_scores(0.2, 1.0, 256) == 278
