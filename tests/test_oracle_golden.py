"""Pin the CPU oracle and the host-side sketch provider against outputs of the
real reference (tests/golden/golden.npz, made by tests/golden/make_golden.py)
and against the SPEC.md known-answer examples.  CPU only."""

import hashlib

import numpy as np
import pytest

from oracle import qjl_oracle as O
from paper_2406_03482_b200 import sketch as SK


# ------------------------------------------------------------- sketch provider
def test_derive_seed_matches_reference(golden):
    for (a, b), want in zip(golden["seed_pairs"], golden["seed_derived"]):
        assert SK.derive_seed(int(a), int(b)) == int(want)


def test_gaussian_bit_identical(golden):
    assert np.array_equal(SK.generate_gaussian(16, 48, 1234).entries, golden["gauss_16x48_1234"])
    big = SK.generate_gaussian(256, 128, SK.derive_seed(0, 0)).entries
    digest = hashlib.sha256(np.ascontiguousarray(big).tobytes()).digest()
    assert digest == golden["gauss_256x128_sha256"].tobytes()


def test_orthogonalize_matches_reference(golden):
    got = SK.orthogonalize(SK.generate_gaussian(300, 64, 9)).entries
    np.testing.assert_allclose(got, golden["orth_300x64_9"], rtol=0, atol=1e-12)
    # rows have norm sqrt(d); rows inside a block are orthogonal (sketch.py:82-103)
    np.testing.assert_allclose(np.linalg.norm(got, axis=1), 8.0, rtol=1e-12)
    blk = got[:64] @ got[:64].T
    np.testing.assert_allclose(blk, 64 * np.eye(64), atol=1e-9)


@pytest.mark.parametrize("m,d", [(0, 4), (4, 0), (-1, 3)])
def test_gaussian_rejects_bad_dims(m, d):
    with pytest.raises(ValueError):
        SK.generate_gaussian(m, d, 0)


# ---------------------------------------------------------------- quantize
def test_quantize_h0_bits_exact(golden):
    r = O.append_keys(golden["q1_S"], None, (), golden["q1_keys"])
    assert np.array_equal(r["bits_in"], golden["q1_bits"])
    np.testing.assert_allclose(r["norm_in"], golden["q1_norm"], rtol=1e-15)
    assert np.all(r["bits_in"][5] == 0xFF) and r["norm_in"][5] == 0.0   # zero key
    assert np.array_equal(r["bits_in"][6], ~r["bits_in"][7])             # sign flip


def test_quantize_outlier_split_bits_exact(golden):
    ch, mags = O.detect_outliers(golden["q2_keys"], 4)
    assert ch == tuple(golden["q2_channels"].tolist())
    np.testing.assert_allclose(mags, golden["q2_mags"], rtol=1e-15)
    r = O.append_keys(golden["q2_S_in"], golden["q2_S_out"], ch, golden["q2_keys"])
    assert np.array_equal(r["bits_in"], golden["q2_bits_in"])
    assert np.array_equal(r["bits_out"], golden["q2_bits_out"])
    np.testing.assert_allclose(r["norm_in"], golden["q2_norm_in"], rtol=1e-15)
    np.testing.assert_allclose(r["norm_out"], golden["q2_norm_out"], rtol=1e-15)
    # fp16 storage policy == reference read_cache semantics
    assert np.array_equal(O.fp16_round(r["norm_in"]), golden["q2_norm_in_f16"])
    assert np.array_equal(O.fp16_round(r["norm_out"]), golden["q2_norm_out_f16"])


def test_logits_and_scores(golden):
    ch = tuple(golden["q2_channels"].tolist())
    cache = O.append_keys(golden["q2_S_in"], golden["q2_S_out"], ch, golden["q2_keys"])
    for i, q in enumerate(golden["q2_queries"]):
        lg = O.estimate_logits(golden["q2_S_in"], golden["q2_S_out"], ch, q, cache)
        np.testing.assert_allclose(lg, golden["q2_logits"][i], rtol=1e-12, atol=1e-12)
        np.testing.assert_allclose(O.softmax(lg), golden["q2_scores_T1"][i], rtol=1e-10, atol=1e-300)
        np.testing.assert_allclose(O.softmax(lg / np.sqrt(128)), golden["q2_scores_Tsqrtd"][i],
                                   rtol=1e-10)
    c16 = dict(cache, norm_in=O.fp16_round(cache["norm_in"]), norm_out=O.fp16_round(cache["norm_out"]))
    for i, q in enumerate(golden["q2_queries"]):
        lg = O.estimate_logits(golden["q2_S_in"], golden["q2_S_out"], ch, q, c16)
        np.testing.assert_allclose(lg, golden["q2_logits_f16norm"][i], rtol=1e-12, atol=1e-12)
    cache1 = O.append_keys(golden["q1_S"], None, (), golden["q1_keys"])
    for i, q in enumerate(golden["q1_queries"]):
        lg = O.estimate_logits(golden["q1_S"], None, (), q, cache1)
        np.testing.assert_allclose(lg, golden["q1_logits"][i], rtol=1e-12, atol=1e-12)


# ------------------------------------------------------------------ values
@pytest.mark.parametrize("b", [1, 2, 3, 8])
def test_value_quantizer_per_token(golden, b):
    v = golden["v_values"]
    codes, zero, scale = O.quantize_values(v, b, group=v.shape[1], const_dtype=None)
    assert np.array_equal(codes, golden[f"v_codes_b{b}"])
    assert np.array_equal(zero[:, 0], golden[f"v_zero_b{b}"])
    assert np.array_equal(scale[:, 0], golden[f"v_scale_b{b}"])
    np.testing.assert_array_equal(O.dequantize_values(codes, zero, scale), golden[f"v_deq_b{b}"])
    assert scale[3, 0] == 0.0 and np.all(codes[3] == 0)   # constant token


def test_quantized_decode(golden):
    ch = tuple(golden["q2_channels"].tolist())
    cache = O.append_keys(golden["q2_S_in"], golden["q2_S_out"], ch, golden["q2_keys"])
    codes, zero, scale = O.quantize_values(golden["dec_values"], 2, 128, const_dtype=None)
    deq = O.dequantize_values(codes, zero, scale)
    for i, q in enumerate(golden["q2_queries"]):
        out, w, _ = O.quantized_decode(golden["q2_S_in"], golden["q2_S_out"], ch, q, cache, deq)
        np.testing.assert_allclose(out, golden["dec_out"][i], rtol=1e-10, atol=1e-12)
        np.testing.assert_allclose(w, golden["dec_weights"][i], rtol=1e-10, atol=1e-300)
        out2, _, _ = O.quantized_decode(golden["q2_S_in"], golden["q2_S_out"], ch, q, cache, deq,
                                        temperature=np.sqrt(128))
        np.testing.assert_allclose(out2, golden["dec_out_Tsqrtd"][i], rtol=1e-10, atol=1e-12)


# ------------------------------------------------------------ edge cases/KATs
def test_detect_outliers_ties(golden):
    assert O.detect_outliers(golden["tie_keys"], 2)[0] == tuple(golden["tie_h2"])
    assert O.detect_outliers(golden["tie_keys"], 3)[0] == tuple(golden["tie_h3"])
    assert O.detect_outliers(golden["tie_keys"], 0)[0] == ()
    assert O.detect_outliers(golden["tie_keys"], 8)[0] == tuple(range(8))
    with pytest.raises(ValueError):
        O.detect_outliers(np.zeros((0, 4)), 1)


def test_pack_non_word_aligned(golden):
    assert np.array_equal(O.pack_rows(golden["pack100_flags"]), golden["pack100_bytes"])
    assert np.array_equal(O.unpack_rows(golden["pack100_bytes"], 100), golden["pack100_flags"])


def test_spec_kats(golden):
    # S = I2, k = (3, -4) -> bits (1, 0), nu = 5
    r = O.quantize_keys(np.eye(2), np.array([[3.0, -4.0]]))
    assert r[0][0, 0] == 0b01 and r[1][0] == 5.0
    assert np.array_equal(r[0][0], golden["kat_qk_bits"])
    # (+,-,+,+,-,-,+,-) -> byte 77
    assert O.pack_rows(np.array([[1, 0, 1, 1, 0, 0, 1, 0]], bool))[0, 0] == 77 == golden["kat_pack_77"][0]
    # sketch_query(I2, (1, 2)) = (1, 2)
    assert np.array_equal(O.sketch_query(np.eye(2), [1.0, 2.0]), [1.0, 2.0])
    # quantize_value((1,2,3), 2) -> zero 1, scale 2/3, codes (0, 2, 3)
    c, z, s = O.quantize_values(np.array([[1.0, 2.0, 3.0]]), 2, 3, const_dtype=None)
    assert np.array_equal(np.array([z[0, 0], s[0, 0], *c[0]]), golden["kat_qv"])
    # SPEC.md:99 / estimator.py:183 -- zero norm -> exactly 0
    lg = O.side_logits(np.eye(2), np.array([1.0, 2.0]), O.pack_rows(np.array([[1, 1]], bool)), [0.0])
    assert lg[0] == 0.0
