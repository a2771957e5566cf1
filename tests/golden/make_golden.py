"""Generate golden vectors by running the REAL reference (pure Python/numpy)
from /root/reference/pkg/src in the build container.

    python tests/golden/make_golden.py      # writes tests/golden/golden.npz

The reference cannot travel to the GPU box, so its outputs are frozen here as
small fixtures.  `tests/test_oracle_golden.py` pins the CPU oracle
(`oracle/qjl_oracle.py`) and the host-side sketch module against them; the
GPU parity tests then compare the device path against the pinned oracle.

Inputs are seeded synthetic tensors (no dataset is involved in this path).
Stream ids follow the reference harness (`pkg/src/qjl/harness.py:38-42`):
keys 0, values 1, queries 2, channels 3.
"""

from __future__ import annotations

import hashlib
import importlib.util
import os
import sys
import tempfile

import numpy as np

REF = "/root/reference/pkg/src/qjl"
OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.npz")


def load_reference():
    spec = importlib.util.spec_from_file_location(
        "qjl_ref", os.path.join(REF, "__init__.py"), submodule_search_locations=[REF])
    mod = importlib.util.module_from_spec(spec)
    sys.modules["qjl_ref"] = mod
    spec.loader.exec_module(mod)
    return mod


def words_to_bytes(words: np.ndarray) -> np.ndarray:
    return np.ascontiguousarray(words, dtype="<u8").view(np.uint8)


def main() -> None:
    ref = load_reference()
    from qjl_ref import estimator as est
    from qjl_ref import kvcache as kv
    from qjl_ref import sketch as rsk
    g: dict[str, np.ndarray] = {}

    # ---------------- sketch module ----------------
    g["seed_pairs"] = np.array([[0, 0], [0, 1], [7, 3], [2**63, 5], [123456789, 2**40]],
                               dtype=np.uint64)
    g["seed_derived"] = np.array([ref.derive_seed(int(a), int(b)) for a, b in g["seed_pairs"]],
                                 dtype=np.uint64)
    g["gauss_16x48_1234"] = ref.generate_gaussian(16, 48, 1234).entries.copy()
    big = ref.generate_gaussian(256, 128, ref.derive_seed(0, 0)).entries
    g["gauss_256x128_sha256"] = np.frombuffer(
        hashlib.sha256(np.ascontiguousarray(big).tobytes()).digest(), np.uint8)
    g["orth_300x64_9"] = ref.orthogonalize(ref.generate_gaussian(300, 64, 9)).entries.copy()

    # ---------------- quantize: C1-shaped unit (h = 0, i.i.d. S) ----------------
    rng = rsk.rng_from_seed(ref.derive_seed(11, 0))
    keys = rng.standard_normal((96, 128)).astype(np.float32).astype(np.float64)
    keys[5] = 0.0                                   # zero key -> all-ones bits, norm 0
    keys[6] = -keys[7]                              # sign-flip pair
    S = ref.generate_gaussian(256, 128, ref.derive_seed(11, 0)).entries
    S = S.astype(np.float32).astype(np.float64)    # any fixed S works; use fp32-rounded
    g["q1_keys"], g["q1_S"] = keys, S
    prof0 = kv.detect_outliers(keys, 0)
    st = kv.KeyCacheState(prof0, ref.SketchMatrix(S, seed=0), None)
    for k in keys:
        st.append(k)
    g["q1_bits"] = np.stack([words_to_bytes(e[0].bits) for e in st.entries])
    g["q1_norm"] = np.array([e[0].norm for e in st.entries])
    q1 = rsk.rng_from_seed(ref.derive_seed(11, 2)).standard_normal((3, 128))
    g["q1_queries"] = q1
    g["q1_logits"] = np.stack([st.estimate_logits(q) for q in q1])

    # ---------------- quantize + logits: C2-shaped unit (h = 4, orthogonal S) ----
    rng = rsk.rng_from_seed(ref.derive_seed(22, 0))
    planted = tuple(sorted(int(c) for c in
                           rsk.rng_from_seed(ref.derive_seed(22, 3)).choice(128, 4, replace=False)))
    keys2 = rng.standard_normal((200, 128))
    keys2[:, list(planted)] *= 15.0
    keys2 = keys2.astype(np.float16).astype(np.float64)
    prof = kv.detect_outliers(keys2, 4)
    assert prof.channels == planted
    st2 = kv.KeyCacheState.create(prof, m_in=256, m_out=128, seed=22)
    for k in keys2:
        st2.append(k)
    g["q2_keys"], g["q2_channels"] = keys2, np.array(prof.channels, np.int32)
    g["q2_mags"] = prof.channel_magnitudes.copy()
    g["q2_S_in"], g["q2_S_out"] = st2.inlier_sketch.entries.copy(), st2.outlier_sketch.entries.copy()
    g["q2_bits_in"] = np.stack([words_to_bytes(e[0].bits) for e in st2.entries])
    g["q2_bits_out"] = np.stack([words_to_bytes(e[1].bits) for e in st2.entries])
    g["q2_norm_in"] = np.array([e[0].norm for e in st2.entries])
    g["q2_norm_out"] = np.array([e[1].norm for e in st2.entries])
    q2 = rsk.rng_from_seed(ref.derive_seed(22, 2)).standard_normal((4, 128))
    g["q2_queries"] = q2
    g["q2_logits"] = np.stack([st2.estimate_logits(q) for q in q2])
    g["q2_scores_T1"] = np.stack([st2.estimate_scores(q).weights for q in q2])
    g["q2_scores_Tsqrtd"] = np.stack([st2.estimate_scores(q, np.sqrt(128)).weights for q in q2])

    # fp16-norm storage semantics: the reference's own write_cache/read_cache
    vals2 = rsk.rng_from_seed(ref.derive_seed(22, 1)).standard_normal((200, 128))
    vtok = [ref.quantize_value(v, 2) for v in vals2]
    with tempfile.TemporaryDirectory() as td:
        path = os.path.join(td, "c.qjlc")
        ref.write_cache(path, st2, vtok)
        st2r, vtok_r, _ = ref.read_cache(path)
    g["q2_norm_in_f16"] = np.array([e[0].norm for e in st2r.entries])
    g["q2_norm_out_f16"] = np.array([e[1].norm for e in st2r.entries])
    g["q2_logits_f16norm"] = np.stack([st2r.estimate_logits(q) for q in q2])

    # ---------------- QJLC cache files (kvcache.py:389-520) ----------------
    # the reference's own write_cache bytes; the device exporter must reproduce them
    # byte for byte from the same keys/values (fp64 keys, per-token values)
    with tempfile.TemporaryDirectory() as td:
        path = os.path.join(td, "c2.qjlc")
        ref.write_cache(path, st2, vtok)
        g["qjlc_c2_bytes"] = np.frombuffer(open(path, "rb").read(), np.uint8).copy()
    # ragged widths: m_in = 96 (2 words, 4 pad bytes), m_out = 40 (partial word)
    # key streams use a master seed other than the sketch seed: keys drawn from the
    # sketch's own stream project to ~0 on an orthogonalized S (sign = rounding noise)
    rng = rsk.rng_from_seed(ref.derive_seed(45, 0))
    k3 = rng.standard_normal((37, 32))
    k3[:, [3, 17, 20, 31]] *= 9.0
    prof3 = kv.detect_outliers(k3, 4)
    st3 = kv.KeyCacheState.create(prof3, m_in=96, m_out=40, seed=44, orthogonalize_sketches=False)
    for k in k3:
        st3.append(k)
    v3 = rsk.rng_from_seed(ref.derive_seed(44, 1)).standard_normal((37, 32))
    v3[2] = 1.25                                     # constant token -> scale 0
    vt3 = [ref.quantize_value(v, 3) for v in v3]
    g["qjlc_r_keys"], g["qjlc_r_values"] = k3, v3
    g["qjlc_r_channels"] = np.array(prof3.channels, np.int32)
    g["qjlc_r_mags"] = prof3.channel_magnitudes.copy()
    # h = 0: no outlier sketch, the record still carries a zero outlier norm
    k4 = rsk.rng_from_seed(ref.derive_seed(56, 0)).standard_normal((9, 64))
    prof4 = kv.detect_outliers(k4, 0)
    st4 = kv.KeyCacheState.create(prof4, m_in=64, seed=55)
    for k in k4:
        st4.append(k)
    v4 = rsk.rng_from_seed(ref.derive_seed(55, 1)).standard_normal((9, 64))
    vt4 = [ref.quantize_value(v, 8) for v in v4]
    g["qjlc_h0_keys"], g["qjlc_h0_values"], g["qjlc_h0_mags"] = k4, v4, prof4.channel_magnitudes.copy()
    with tempfile.TemporaryDirectory() as td:
        for name, st_, vt_ in (("r", st3, vt3), ("h0", st4, vt4)):
            path = os.path.join(td, name + ".qjlc")
            ref.write_cache(path, st_, vt_)
            g[f"qjlc_{name}_bytes"] = np.frombuffer(open(path, "rb").read(), np.uint8).copy()
            st_r, _, _ = ref.read_cache(path)
            qs = rsk.rng_from_seed(ref.derive_seed(66, 2)).standard_normal((2, st_.d))
            g[f"qjlc_{name}_queries"] = qs
            g[f"qjlc_{name}_logits"] = np.stack([st_r.estimate_logits(q) for q in qs])
            g[f"qjlc_{name}_out"] = np.stack(
                [ref.quantized_decode(q, st_r, ref.read_cache(path)[1]).output for q in qs])

    # ---------------- statistical suites (harness.py:183-329) ----------------
    from qjl_ref import harness as hz
    suites = {
        "unb_sphere": ("run_unbiasedness_trial", dict(d=64, m=8, trials=300, seed=3, distribution="sphere")),
        "unb_outlier_iid": ("run_unbiasedness_trial", dict(d=32, m=16, trials=200, seed=4,
                                                           distribution="outlier", orthogonalize=False)),
        "dist_m64": ("run_distortion_trial", dict(d=64, m=64, trials=300, seed=5, distribution="gaussian")),
        "dist_m8": ("run_distortion_trial", dict(d=64, m=8, trials=300, seed=5, distribution="gaussian")),
        "scores": ("run_score_trial", dict(d=32, m=64, n=64, trials=100, seed=6)),
        "orth": ("run_orthogonal_comparison", dict(d=64, m=16, trials=300, seed=7)),
    }
    fields = ["passed", "trials", "mean_estimate", "true_value", "stderr", "z_score", "failure_fraction",
              "threshold", "fraction_within_bound", "variance_ratio", "score_err_p50", "score_err_p90",
              "score_err_p99", "score_err_max"]
    g["harness_fields"] = np.array(fields)
    for name, (fn, kw) in suites.items():
        row = getattr(hz, fn)(hz.TrialConfig(**kw)).to_row()
        g[f"harness_{name}"] = np.array([np.nan if row.get(f) is None else float(row[f]) for f in fields])

    # ---------------- values (per-token, reference semantics) ----------------
    vals = rsk.rng_from_seed(ref.derive_seed(33, 1)).standard_normal((64, 32))
    vals[3] = 5.0                                    # constant token -> scale 0
    vals[4] = np.array([0.0, 1.0, 2.0, 3.0] * 8) / 3.0  # exact .5 ties under b=1
    g["v_values"] = vals
    for b in (1, 2, 3, 8):
        toks = [ref.quantize_value(v, b) for v in vals]
        g[f"v_codes_b{b}"] = np.stack([t.codes for t in toks])
        g[f"v_zero_b{b}"] = np.array([t.zero for t in toks])
        g[f"v_scale_b{b}"] = np.array([t.scale for t in toks])
        g[f"v_deq_b{b}"] = np.stack([ref.dequantize_value(t) for t in toks])

    # ---------------- quantized_decode (reference per-token values) ----------
    dec_out, dec_w = [], []
    for q in q2:
        r = ref.quantized_decode(q, st2, vtok, temperature=1.0)
        dec_out.append(r.output)
        dec_w.append(r.scores.weights)
    g["dec_values"] = vals2
    g["dec_out"], g["dec_weights"] = np.stack(dec_out), np.stack(dec_w)
    g["dec_out_Tsqrtd"] = np.stack(
        [ref.quantized_decode(q, st2, vtok, temperature=np.sqrt(128)).output for q in q2])

    # ---------------- detect_outliers: ties + degenerate h ----------------
    tie = np.ones((5, 8))
    tie[:, 2] = 3.0
    tie[:, 6] = 3.0
    tie[:, 4] = -3.0
    g["tie_keys"] = tie
    g["tie_h2"] = np.array(kv.detect_outliers(tie, 2).channels, np.int32)
    g["tie_h3"] = np.array(kv.detect_outliers(tie, 3).channels, np.int32)

    # ---------------- packing with m not a multiple of 64 ----------------
    flags = rsk.rng_from_seed(5).integers(0, 2, size=(10, 100)).astype(bool)
    g["pack100_flags"] = flags
    g["pack100_bytes"] = np.stack([words_to_bytes(est._pack_bool(f)) for f in flags])

    # ---------------- SPEC known-answer tests ----------------
    I2 = ref.SketchMatrix(np.eye(2), seed=0)
    qk = ref.quantize_key(I2, np.array([3.0, -4.0]))
    g["kat_qk_bits"] = words_to_bytes(qk.bits)
    g["kat_qk_norm"] = np.array(qk.norm)
    g["kat_pack_77"] = words_to_bytes(ref.pack_signs(np.array([1, -1, 1, 1, -1, -1, 1, -1])))
    qv = ref.quantize_value(np.array([1.0, 2.0, 3.0]), 2)
    g["kat_qv"] = np.array([qv.zero, qv.scale, *qv.codes.astype(np.float64)])
    g["kat_required_m"] = np.array([ref.required_m(0.25, 0.01),
                                    ref.required_m_scores(0.2, 1.0, 256)])

    np.savez_compressed(OUT, **g)
    print(f"wrote {OUT} ({os.path.getsize(OUT)} bytes, {len(g)} arrays)")


if __name__ == "__main__":
    main()
