"""Statistical suites on the B200: the batched device harness
reproduces the real reference harness's reports (tests/golden), and the device
orthogonalization (qjl_orthogonalize) matches sketch.py:82-103."""

import numpy as np
import pytest
import torch

from paper_2406_03482_b200 import harness as H
from paper_2406_03482_b200 import sketch as SK
from tests.test_harness_cpu import SUITES, check_report

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("m,d", [(8, 64), (300, 64), (256, 128), (16, 32), (100, 100), (5, 3)])
def test_device_orthogonalize_matches_reference(cuda, m, d):
    G = np.stack([SK.generate_gaussian(m, d, s).entries for s in range(6)])
    got = H.orthogonalize_batch(G).cpu().numpy()
    for i in range(6):
        want = SK.orthogonalize(SK.SketchMatrix(G[i], seed=0)).entries
        np.testing.assert_allclose(got[i], want, rtol=0, atol=1e-12)


@pytest.mark.parametrize("name", sorted(SUITES))
def test_device_suites_reproduce_reference_reports(cuda, golden, name):
    fn, kw = SUITES[name]
    row = getattr(H, fn)(H.TrialConfig(**kw)).to_row()
    # f32 sign-dot sums on the device: means / variances agree to ~1e-6 relative
    check_report(row, golden[f"harness_{name}"], golden["harness_fields"], rtol=2e-5, ztol=2e-3)


def test_full_size_unbiasedness_passes(cuda):
    """The reference's default suite size (10000 sketches, d = 64, m = 8) in one batch."""
    r = H.run_unbiasedness_trial(H.TrialConfig())
    assert r.passed and abs(r.z_score) <= H.MEAN_Z_BOUND
    o = H.run_orthogonal_comparison(H.TrialConfig(trials=2000))
    assert o.passed and o.variance_ratio <= H.VARIANCE_RATIO_BOUND
