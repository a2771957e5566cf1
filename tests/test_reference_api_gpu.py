"""The drop-in API (paper_2406_03482_b200 mirrors of pkg/src/qjl) on the B200,
checked against the golden outputs of the real reference (tests/golden) and the
SPEC.md known answers -- written like the reference's own tests would be."""

import numpy as np
import pytest

import paper_2406_03482_b200 as qjl
from oracle import qjl_oracle as O

pytestmark = pytest.mark.gpu


def _words(golden_bytes):
    return np.ascontiguousarray(golden_bytes).view("<u8")


def test_spec_kats(cuda, golden):
    I2 = qjl.SketchMatrix(np.eye(2), seed=0)
    qk = qjl.quantize_key(I2, np.array([3.0, -4.0]))
    assert np.array_equal(np.ascontiguousarray(qk.bits).view(np.uint8), golden["kat_qk_bits"])
    assert qk.norm == 5.0 and qk.m == 2
    zk = qjl.quantize_key(I2, np.zeros(2))
    assert int(zk.bits[0]) == 0b11 and zk.norm == 0.0
    sq = qjl.sketch_query(I2, np.array([1.0, 2.0]))
    assert np.array_equal(sq.values, [1.0, 2.0])
    assert qjl.estimate_inner_product(sq, zk) == 0.0
    assert np.array_equal(np.ascontiguousarray(qjl.pack_signs(np.array([1, -1, 1, 1, -1, -1, 1, -1]))).view(np.uint8)[:1],
                          golden["kat_pack_77"][:1])
    qv = qjl.quantize_value(np.array([1.0, 2.0, 3.0]), 2)
    assert list(qv.codes) == [0, 2, 3] and qv.zero == 1.0
    assert abs(qv.scale - 2.0 / 3.0) < 1e-7
    cv = qjl.quantize_value(np.array([5.0, 5.0, 5.0]), 3)
    assert cv.scale == 0.0 and list(cv.codes) == [0, 0, 0]
    prof = qjl.detect_outliers(np.tile([1.0, 1.0, 10.0, 1.0], (3, 1)), 1)
    assert prof.channels == (2,)
    p2 = qjl.OutlierProfile(channels=(1,), d=2, channel_magnitudes=np.zeros(2))
    a, b = p2.split(np.array([3.0, -4.0]))
    assert a.tolist() == [3.0] and b.tolist() == [-4.0]
    with pytest.raises(ValueError):
        qjl.quantize_key(I2, np.zeros(3))
    with pytest.raises(ValueError):
        qjl.estimate_inner_product(qjl.sketch_query(I2, [1.0, 0.0]),
                                   qjl.QuantizedKey(bits=np.zeros(1, "<u8"), norm=1.0, m=3))


def test_key_cache_state_matches_reference_h0(cuda, golden):
    """Config-1 shaped unit: bits exact, logits within the north-star tolerance."""
    prof = qjl.detect_outliers(golden["q1_keys"], 0)
    st = qjl.KeyCacheState(prof, qjl.SketchMatrix(golden["q1_S"], seed=0), None)
    for k in golden["q1_keys"][:10]:
        st.append(k)                                             # single-key appends
    st.extend(golden["q1_keys"][10:])                            # batched append
    assert st.n == golden["q1_keys"].shape[0]
    ent = st.entries
    for i, (ki, ko) in enumerate(ent):
        assert np.array_equal(np.ascontiguousarray(ki.bits).view(np.uint8), golden["q1_bits"][i])
        assert ki.norm == golden["q1_norm"][i]                   # fp64 ||k||, as quantize_key returns
        assert ko.m == 0
    for i, q in enumerate(golden["q1_queries"]):
        lg = st.estimate_logits(q)
        ref = golden["q1_logits"][i]
        assert np.all(np.abs(lg - ref) <= 1e-3 * np.abs(ref) + 1e-4), np.abs(lg - ref).max()


def test_key_cache_state_outliers_scores_and_decode(cuda, golden):
    """Config-2 shaped unit (h = 4, orthogonal S from the reference seed)."""
    prof = qjl.detect_outliers(golden["q2_keys"], 4)
    assert prof.channels == tuple(golden["q2_channels"].tolist())
    np.testing.assert_allclose(prof.channel_magnitudes, golden["q2_mags"], rtol=1e-14)
    st = qjl.KeyCacheState.create(prof, m_in=256, m_out=128, seed=22)
    np.testing.assert_array_equal(st.inlier_sketch.entries, golden["q2_S_in"])
    st.extend(golden["q2_keys"])
    ent = st.entries
    for i, (ki, ko) in enumerate(ent):
        assert np.array_equal(np.ascontiguousarray(ki.bits).view(np.uint8), golden["q2_bits_in"][i])
        assert np.array_equal(np.ascontiguousarray(ko.bits).view(np.uint8), golden["q2_bits_out"][i])
        assert ki.norm == golden["q2_norm_in"][i] and ko.norm == golden["q2_norm_out"][i]
    for i, q in enumerate(golden["q2_queries"]):
        lg = st.estimate_logits(q)
        ref = golden["q2_logits_f16norm"][i]     # reference state with fp16-stored norms
        assert np.all(np.abs(lg - ref) <= 1e-3 * np.abs(ref) + 1e-4)
        sc = st.estimate_scores(q)
        assert abs(sc.weights.sum() - 1.0) <= 1e-6
        ref_w = O.softmax(ref)
        assert np.abs(sc.weights - ref_w).sum() <= 2e-3          # TV distance of the scores
    # decode: reference semantics with the fp16 norm storage policy (oracle pinned to
    # the reference in tests/test_oracle_golden.py)
    vtok = [qjl.quantize_value(v, 2) for v in golden["dec_values"]]
    codes, zero, scale = O.quantize_values(golden["dec_values"], 2, 128, const_dtype=None)
    deq = O.dequantize_values(codes, zero, scale)
    cache = O.append_keys(golden["q2_S_in"], golden["q2_S_out"], prof.channels, golden["q2_keys"])
    cache["norm_in"], cache["norm_out"] = O.fp16_round(cache["norm_in"]), O.fp16_round(cache["norm_out"])
    for i, q in enumerate(golden["q2_queries"]):
        for T in (1.0, float(np.sqrt(128))):
            r = qjl.quantized_decode(q, st, vtok, temperature=T)
            ref, _, _ = O.quantized_decode(golden["q2_S_in"], golden["q2_S_out"], prof.channels, q,
                                           cache, deq, T)
            assert np.linalg.norm(r.output - ref) / np.linalg.norm(ref) <= 1e-3
            assert abs(r.scores.weights.sum() - 1.0) <= 1e-6
    with pytest.raises(ValueError):
        qjl.quantized_decode(golden["q2_queries"][0], st, vtok[:-1])
    with pytest.raises(ValueError):
        st.estimate_scores(golden["q2_queries"][0], temperature=0.0)


def test_value_quantizer_matches_reference(cuda, golden):
    v = golden["v_values"]
    for b in (1, 2, 3, 8):
        toks = [qjl.quantize_value(row, b) for row in v]
        assert np.array_equal(np.stack([t.codes for t in toks]), golden[f"v_codes_b{b}"])
        np.testing.assert_allclose([t.zero for t in toks], golden[f"v_zero_b{b}"], rtol=1e-7)
        np.testing.assert_allclose([t.scale for t in toks], golden[f"v_scale_b{b}"], rtol=1e-7)


@pytest.mark.parametrize("m", [1, 7, 64, 100, 130, 512])
def test_packed_kernel_equals_naive_pm1(cuda, m):
    """SPEC acceptance 4: packed kernel == naive +/-1 loop within 1e-5 relative,
    m in 1..512 including non-word-aligned sizes."""
    rng = np.random.default_rng(m)
    for _ in range(5):
        signs = np.where(rng.random(m) < 0.5, -1, 1)
        vals = rng.standard_normal(m)
        words = qjl.pack_signs(signs)
        assert np.array_equal(qjl.unpack_signs(words, m), signs)
        got = qjl.packed_sign_dot(vals, words, m)
        ref = float(np.dot(vals, signs))
        assert abs(got - ref) <= 1e-5 * max(1.0, abs(ref))


def test_non_aligned_sketch_width(cuda):
    """m = 100 (not a multiple of 32): logits still use sqrt(pi/2)/m with the true m."""
    rng = np.random.default_rng(1)
    S = qjl.generate_gaussian(100, 16, 5)
    prof = qjl.OutlierProfile(channels=(), d=16, channel_magnitudes=np.zeros(16))
    st = qjl.KeyCacheState(prof, S, None)
    keys = rng.standard_normal((40, 16))
    st.extend(keys)
    q = rng.standard_normal(16)
    sq = qjl.sketch_query(S, q)
    ref = np.array([qjl.ESTIMATOR_SCALE / 100 * float(np.float16(np.linalg.norm(k))) *
                    float(np.dot(sq.values, np.where(S.entries @ k >= 0, 1.0, -1.0))) for k in keys])
    np.testing.assert_allclose(st.estimate_logits(q), ref, rtol=1e-4, atol=1e-5)
    for (ki, _), k in zip(st.entries, keys):
        assert np.array_equal(qjl.unpack_signs(ki.bits, 100), np.where(S.entries @ k >= 0, 1, -1))
