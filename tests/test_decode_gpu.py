"""Tensor-core decode and scores (csrc/k_decode.cu, tile-major P2T records) against the CPU
oracle: stream-K unit boundaries and tail tiles, head counts 1/2/3/4, every sketch width
the kernels instantiate, temperature 1 and sqrt(d), log-sum-exp, the scores-only kernel,
the P2T value quantizer, determinism and the decode-kernel benchmark hook."""

import numpy as np
import pytest
import torch

from oracle import qjl_oracle as O
from tests._cache import logsumexp, make_cache, oracle_decode
from tests._parity import OUT_RTOL, check_logits, logit_bound, rel_l2

pytestmark = pytest.mark.gpu

SHAPES = [
    # U, n, G, h, m_in, m_out
    (64, 4096, 4, 8, 256, 64),      # many CTAs per unit, segments cross units
    (8, 100, 4, 8, 256, 64),        # fewer tiles than CTAs, tail tile
    (3, 1, 2, 8, 256, 64),          # n = 1
    (16, 2000, 1, 4, 256, 128),     # MHA, config-2 sketch sizes
    (4, 3000, 4, 0, 256, 0),        # no outliers
    (4, 3000, 3, 8, 512, 64),       # m = 512, G = 3
    (8, 5000, 2, 8, 256, 64),       # G = 2 (two-head epilogue)
    (6, 2500, 1, 8, 512, 64),       # G = 1 with m = 512
    (4, 1500, 4, 4, 512, 128),      # m = 512 + 128
    (4, 1300, 4, 0, 512, 0),        # m = 512, no outliers
]


def _sample_units(U):
    return sorted({0, U // 2, U - 1})


@pytest.mark.parametrize("U,n,G,h,m_in,m_out", SHAPES)
def test_decode_matches_oracle(cuda, U, n, G, h, m_in, m_out):
    c, q = make_cache(U, n, G, h, m_in, m_out, seed=U * 7 + n)
    assert c.tensor_core_path(G)
    for T in (1.0, float(np.sqrt(128))):
        lse = torch.empty(U, G, device="cuda")
        out = c.decode(q, temperature=T, lse=lse).double().cpu().numpy()
        lse = lse.double().cpu().numpy()
        assert np.isfinite(out).all()
        for u in _sample_units(U):
            ref, logits = oracle_decode(c, q, u, T)
            ref_lse = logsumexp(logits / T)
            for g in range(G):
                e = rel_l2(out[u, g], ref[g])
                assert e <= OUT_RTOL, (u, g, T, e)
                # the fused kernel's own log-sum-exp against the oracle's logits
                assert abs(lse[u, g] - ref_lse[g]) <= 1e-4 * max(1.0, abs(ref_lse[g])), (u, g, T)


@pytest.mark.parametrize("U,n,G,h,m_in,m_out", [SHAPES[0], SHAPES[1], SHAPES[3], SHAPES[4], SHAPES[5],
                                                 (2, 700, 1, 0, 256, 0)])
def test_scores_kernel_matches_oracle(cuda, U, n, G, h, m_in, m_out):
    """Scores-only K2 on tile records (kvcache.py:311-329) against estimate_logits."""
    c, q = make_cache(U, n, G, h, m_in, m_out, seed=U + 3 * n)
    assert c.tensor_core_path(G, scores=True)
    logits = c.scores(q).double().cpu().numpy()
    from tests._cache import oracle_unit

    Qh = q.double().cpu().numpy()
    for u in _sample_units(U):
        chans, cache, _ = oracle_unit(c, u)
        for g in range(G):
            ref = O.estimate_logits(c.S_in_host, c.S_out_host, chans, Qh[u, g], cache)
            ok, err = check_logits(logits[u, g], ref,
                                   logit_bound(c.S_in_host, c.S_out_host, chans, Qh[u, g], cache["norm_in"],
                                               cache.get("norm_out", 0.0)))
            assert ok.all(), (u, g, err.max())


def test_full_config3_against_oracle(cuda):
    """Full config-3 shape (64 units x 32768 tokens, 4 q-heads/unit); the oracle checks
    the first and last units."""
    U, n, G = 64, 32768, 4
    c, q = make_cache(U, n, G, 8, 256, 64, seed=3)
    lse = torch.empty(U, G, device="cuda")
    out = c.decode(q, lse=lse).double().cpu().numpy()
    assert np.isfinite(out).all()
    for u in (0, U - 1):
        ref, logits = oracle_decode(c, q, u)
        ref_lse = logsumexp(logits)
        for g in range(G):
            assert rel_l2(out[u, g], ref[g]) <= OUT_RTOL, (u, g, rel_l2(out[u, g], ref[g]))
            assert abs(float(lse[u, g]) - ref_lse[g]) <= 1e-4 * abs(ref_lse[g])


def _close(a, b, tol=1e-5):
    a, b = a.double(), b.double()
    return float((a - b).norm() / b.norm().clamp_min(1e-300)) <= tol


def test_determinism_and_chaining(cuda):
    """Both schedules are bitwise reproducible run to run (fixed partial slots, fixed merge
    order); they differ from each other only in rounding (different segmentations)."""
    c, q = make_cache(8, 5000, 4, 8, 256, 64, seed=11)
    d1 = c.decode(q, deterministic=True).clone()
    d2 = c.decode(q, deterministic=True, chained=True).clone()
    d3 = c.decode(q, deterministic=True, chained=True)
    assert torch.equal(d1, d2) and torch.equal(d1, d3)
    o1 = c.decode(q).clone()
    o2 = c.decode(q, chained=True).clone()       # PDL-chained on the previous decode
    o3 = c.decode(q, chained=True)
    assert torch.equal(o1, o2) and torch.equal(o1, o3)
    assert _close(o1, d1)


def test_replica_decodes_identically(cuda):
    """DeviceKeyCache.replica(): same contents in its own record buffer (bench.py rotates
    steps over replicas so sub-L2 shards are read from HBM); decodes and logits are bitwise
    those of the original, also chained across replicas, and writes do not alias."""
    c, q = make_cache(8, 3000, 4, 8, 256, 64, seed=5)
    r = c.replica()
    assert r.records.data_ptr() != c.records.data_ptr() and torch.equal(r.records, c.records)
    assert r.key_desc().bits_in != c.key_desc().bits_in
    o = c.decode(q).clone()
    o1 = r.decode(q, chained=True).clone()
    o2 = c.decode(q, chained=True).clone()
    assert torch.equal(o, o1) and torch.equal(o, o2)
    assert torch.equal(c.scores(q), r.scores(q))
    r.records.zero_()
    assert torch.equal(c.decode(q), o)


def test_decode_captures_into_a_cuda_graph(cuda):
    """The launch path allocates nothing and synchronises nothing once its workspace exists,
    so a serving loop can capture chained decode steps (their PDL edges included) in one
    CUDA graph; the replay is bitwise the eager result and follows new query contents."""
    c, q = make_cache(8, 3000, 4, 8, 256, 64, seed=9)
    out = torch.empty(8, 4, 128, device="cuda")
    ref = c.decode(q).clone()                       # also sizes the workspace
    gq = q.clone()
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        c.decode(gq, out=out)
    torch.cuda.current_stream().wait_stream(side)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for i in range(3):
            c.decode(gq, out=out, chained=i > 0)
    out.zero_()
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(out, ref)
    q2 = torch.randn_like(q.float()).to(q.dtype)
    gq.copy_(q2)
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(out, c.decode(q2))


def test_scores_chaining(cuda):
    """qjl_scores with QJL_DECODE_CHAINED (PDL: the query sketch overlaps the previous score
    or decode kernel) writes the same logits as unchained calls, including after a decode
    and with a different query (the previous kernel still reads the workspace)."""
    c, q = make_cache(8, 5000, 4, 8, 256, 64, seed=12)
    q2 = torch.flip(q, dims=[0]).contiguous()
    l1 = c.scores(q).clone()
    m1 = c.scores(q2).clone()
    l2 = c.scores(q, chained=True).clone()
    m2 = c.scores(q2, chained=True).clone()
    c.decode(q)
    l3 = c.scores(q, chained=True).clone()
    m3 = c.scores(q2, chained=True)
    assert torch.equal(l1, l2) and torch.equal(l1, l3)
    assert torch.equal(m1, m2) and torch.equal(m1, m3)
    assert not torch.equal(l1, m1)


def test_bench_hook_runs_the_same_kernel(cuda):
    c, q = make_cache(16, 3000, 4, 8, 256, 64, seed=5)
    ref = c.decode(q).clone()
    out = torch.empty_like(ref)
    ms = c.bench_decode_kernel(q, reps=5, out=out)
    assert ms > 0
    assert torch.equal(out, ref)                 # every chained kernel rewrites the same output
    assert torch.equal(c.decode(q), ref)         # counters were left clean
    out.zero_()
    c.bench_decode_kernel(q, reps=3, out=out, deterministic=True)
    assert torch.equal(out, c.decode(q, deterministic=True))


def test_p2t_codes_match_oracle_quantizer(cuda):
    from paper_2406_03482_b200.device import DeviceKeyCache, unpack_codes

    U, n = 3, 300
    V = torch.randn(U, n, 128, device="cuda", dtype=torch.bfloat16)
    c = DeviceKeyCache(U, 128, 256, 0, 0, n)
    c.append_values(V)
    Vh = V.double().cpu().numpy()
    for u in range(U):
        codes, zero, scale = O.quantize_values(Vh[u], 2, 32)
        assert np.array_equal(unpack_codes(c.v_codes[u].cpu().numpy(), n), codes)
        assert np.array_equal(c.v_zero[u, :n].double().cpu().numpy(), zero)
        assert np.array_equal(c.v_scale[u, :n].double().cpu().numpy(), scale)


def test_p2t_quantizer_exact_ties_and_unaligned_appends(cuda):
    """Values on a grid that puts many quotients exactly on .5 (round-half-even in the
    reference), constant groups, and appends starting at rows that are not multiples of 4."""
    from paper_2406_03482_b200.device import DeviceKeyCache, unpack_codes

    U, n = 2, 203
    g = torch.Generator().manual_seed(5)
    V = (torch.randint(0, 7, (U, n, 128), generator=g).double() * 0.5)   # multiples of 1/2 -> ties
    V[:, 7, 32:64] = 1.25                                                   # constant group
    V[:, 11] *= 1e-3
    Vt = V.to(torch.bfloat16)
    c = DeviceKeyCache(U, 128, 256, 0, 0, n)
    for a, b in ((0, 5), (5, 6), (6, 70), (70, 203)):                       # unaligned row offsets
        c.append_values(Vt[:, a:b].to(cuda))
    Vh = Vt.double().numpy()
    for u in range(U):
        codes, zero, scale = O.quantize_values(Vh[u], 2, 32, const_dtype="f16")
        assert np.array_equal(unpack_codes(c.v_codes[u].cpu().numpy(), n), codes)
        assert np.array_equal(c.v_zero[u, :n].double().cpu().numpy(), zero)
        assert np.array_equal(c.v_scale[u, :n].double().cpu().numpy(), scale)


def test_stale_padding_rows_are_masked(cuda):
    """Rows >= n of the last tile hold garbage (NaN/Inf constants, random bits): the
    decode must ignore them (the masked tail tile zeroes their constants)."""
    c, q = make_cache(4, 1000, 4, 8, 256, 64, seed=17, capacity=1024)
    ref = c.decode(q, deterministic=True).clone()
    rows = slice(1000, 1024)
    for name, val in (("v_scale", float("inf")), ("v_zero", float("nan")), ("norm_in", float("nan")),
                      ("bits_in", 0x55)):
        c.fill_rows(name, rows, val)
    # P2T codes are tile-interleaved: the bytes of tokens 1000..1023 (tile 7, rows 104..127)
    from paper_2406_03482_b200.device import _P2T_BYTE

    fv = c.field_view("v_codes")
    flat = fv.view(fv.shape[0], fv.shape[1], 4096)
    idx = torch.as_tensor(np.unique(_P2T_BYTE[104:128].ravel()), device="cuda")
    flat[:, 7, idx] = 0xFF
    out = c.decode(q, deterministic=True)
    assert torch.equal(out, ref)


def test_rejects_unsupported_p2t_shapes(cuda):
    from paper_2406_03482_b200.device import DeviceKeyCache

    c = DeviceKeyCache(2, 128, 256, 0, 0, 256)
    c.set_sketches(*DeviceKeyCache.make_sketches(128, 0, 256, 0, operand="bf16"))
    K = torch.randn(2, 10, 128, device="cuda", dtype=torch.bfloat16)
    c.append(K, K)
    assert c.tensor_core_path(4) and not c.tensor_core_path(5)
    with pytest.raises(NotImplementedError):
        c.decode(torch.randn(2, 5, 128, device="cuda", dtype=torch.bfloat16))   # G = 5 > 4


def test_sharded_decode_bitwise_equals_full(cuda):
    """units are independent, so decoding the unit range a rank owns
    (KV-head shards of config 3 at 2/4/8 GPUs) gives the unsharded decode's rows bit for bit
    under the deterministic schedule (fixed 512-token segments), and within rounding under
    the default stream-K schedule; the shard's cache records are the full cache's."""
    import bench
    from paper_2406_03482_b200.distributed import shard_units

    w = dict(bench.WORKLOADS["c3"], n=4096)            # 64 units x 32 tiles, 8 segments per unit
    one = shard_units(64, 1, 0)
    full = bench.build_cache(w, one, 5, cuda)
    qf = bench.make_queries(w, one, 5, cuda)
    of = full.decode(qf, deterministic=True).clone()
    od = full.decode(qf).clone()
    ref, _ = oracle_decode(full, qf, 63)
    for g in range(4):
        assert rel_l2(of[63, g].double().cpu().numpy(), ref[g]) <= OUT_RTOL
    for world in (2, 4, 8):
        for r in sorted({0, world // 2, world - 1}):
            sh = shard_units(64, world, r)
            c = bench.build_cache(w, sh, 5, cuda)
            q = bench.make_queries(w, sh, 5, cuda)
            assert torch.equal(q, qf[sh.start:sh.stop])
            assert torch.equal(c.records, full.records[sh.start:sh.stop])
            o = c.decode(q, deterministic=True)
            assert torch.equal(o, of[sh.start:sh.stop]), (world, r)
            o2 = c.decode(q).double()
            e = (o2 - od[sh.start:sh.stop].double()).norm() / od[sh.start:sh.stop].double().norm()
            assert e <= 1e-5, (world, r, float(e))


def test_full_config2_against_oracle(cuda):
    """Full config-2 shape: Llama-2-7B MHA decode, 4 x 32 = 128 units x 4096 tokens, fp16,
    h = 4 outlier channels x15, m_in 256 + m_out 128; decode, lse and the scores kernel on
    sampled units against the oracle."""
    U, n, G = 128, 4096, 1
    c, q = make_cache(U, n, G, 4, 256, 128, seed=2, dtype=torch.float16, factor=15.0)
    assert c.tensor_core_path(G) and c.tensor_core_path(G, scores=True)
    lse = torch.empty(U, G, device="cuda")
    out = c.decode(q, lse=lse).double().cpu().numpy()
    logits = c.scores(q).double().cpu().numpy()
    from tests._cache import oracle_unit

    Qh = q.double().cpu().numpy()
    for u in (0, 61, U - 1):
        ref, ref_lg = oracle_decode(c, q, u)
        assert rel_l2(out[u, 0], ref[0]) <= OUT_RTOL
        assert abs(float(lse[u, 0]) - logsumexp(ref_lg)[0]) <= 1e-4 * abs(logsumexp(ref_lg)[0])
        chans, cache, _ = oracle_unit(c, u)
        ok, err = check_logits(logits[u, 0], ref_lg[0],
                               logit_bound(c.S_in_host, c.S_out_host, chans, Qh[u, 0], cache["norm_in"],
                                           cache["norm_out"]))
        assert ok.all(), (u, err.max())


@pytest.mark.parametrize("B,n", [(2, 32768), (1, 131072)])
def test_config5_m512_long_context_against_oracle(cuda, B, n):
    """Config 5 with m = 512 (+ m_out 64, r = 8 x20) at n >= 32k: B x 8 KV-head units, G = 4;
    the first and last units against the oracle."""
    U, G = B * 8, 4
    c, q = make_cache(U, n, G, 8, 512, 64, seed=B + n)
    assert c.tensor_core_path(G)
    lse = torch.empty(U, G, device="cuda")
    out = c.decode(q, lse=lse).double().cpu().numpy()
    for u in (0, U - 1):
        ref, lg = oracle_decode(c, q, u)
        ref_lse = logsumexp(lg)
        for g in range(G):
            assert rel_l2(out[u, g], ref[g]) <= OUT_RTOL, (u, g, rel_l2(out[u, g], ref[g]))
            assert abs(float(lse[u, g]) - ref_lse[g]) <= 1e-4 * abs(ref_lse[g])
