"""Host-side layout logic of the tile-major cache (no GPU): the P2T code layout is a
bijection whose 16-byte chunks are swizzled so that the 8 dim quads a warp reads sit in
8 different bank groups, and pack/unpack round-trip (csrc/common.cuh p2t_byte)."""

import numpy as np

from paper_2406_03482_b200.device import _P2T_BYTE, _P2T_SHIFT, pack_codes, unpack_codes


def test_p2t_layout_is_a_bijection():
    pairs = _P2T_BYTE.astype(np.int64) * 8 + _P2T_SHIFT
    assert len(np.unique(pairs)) == 128 * 128
    assert _P2T_BYTE.min() == 0 and _P2T_BYTE.max() == 4095


def test_p2t_word_holds_four_tokens_of_four_dims():
    # the decode masks one u32 word per (dim, 4-token group): bytes of a word = 4 tokens
    for t0 in range(0, 128, 4):
        for d0 in range(0, 128, 4):
            words = {int(b) // 4 for b in _P2T_BYTE[t0:t0 + 4, d0:d0 + 4].ravel()}
            assert len(words) == 1


def test_p2t_chunks_conflict_free_per_phase():
    # a 128-bit shared load is served 8 threads at a time; threads 8p..8p+7 = two dim quads,
    # whose 16-byte chunks j must fall in different 16-byte bank groups (address / 16 mod 8)
    for dq in range(0, 32, 2):
        for j in range(8):
            tok = 16 * j
            a, b = int(_P2T_BYTE[tok, 4 * dq]), int(_P2T_BYTE[tok, 4 * dq + 4])
            assert (a // 16) % 8 != (b // 16) % 8


def test_pack_unpack_round_trip():
    rng = np.random.default_rng(3)
    for n in (1, 127, 128, 300):
        codes = rng.integers(0, 4, (2, n, 128)).astype(np.uint8)
        packed = pack_codes(codes)
        assert packed.shape == (2, (n + 127) // 128 * 128, 32)
        assert np.array_equal(unpack_codes(packed, n), codes)
