"""Host-side sketch provider: seeded Gaussian JL matrices, seed derivation and
blockwise row orthogonalization.

This is one-time setup, not the hot path: the reference draws S on the host
(`pkg/src/qjl/sketch.py:66-103`) and so do we; the device receives S once,
rounded to the MMA operand dtype and laid out per unit (see
`DeviceKeyCache.set_sketches`).

Algorithms restated (not copied) from the reference:
  * `derive_seed`  -- SplitMix64 finalizer over master + GAMMA*(stream+1)
                      (`pkg/src/qjl/sketch.py:19-32`).
  * `rng_from_seed` -- numpy Philox keyed by the 64-bit seed
                      (`pkg/src/qjl/sketch.py:35-37`).
  * `generate_gaussian` -- standard_normal((m, d)) from that generator
                      (`pkg/src/qjl/sketch.py:66-79`).
  * `orthogonalize` -- QR per block of <= d rows of ONE draw, sign-fixed by
                      diag(R) (0 -> +1), rows rescaled to sqrt(d)
                      (`pkg/src/qjl/sketch.py:82-103`).
numpy's Generator stream is version dependent, so S is always generated
in-process and never hard-coded.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

_U64 = (1 << 64) - 1
_SPLITMIX_GAMMA = 0x9E3779B97F4A7C15
_SPLITMIX_M1 = 0xBF58476D1CE4E5B9
_SPLITMIX_M2 = 0x94D049BB133111EB


def derive_seed(master: int, stream: int) -> int:
    """SplitMix64 finalizer of ``master + GAMMA * (stream + 1)`` (mod 2^64)."""
    z = (int(master) + _SPLITMIX_GAMMA * (int(stream) + 1)) & _U64
    for shift, mult in ((30, _SPLITMIX_M1), (27, _SPLITMIX_M2)):
        z = ((z ^ (z >> shift)) * mult) & _U64
    return z ^ (z >> 31)


def rng_from_seed(seed: int) -> np.random.Generator:
    """numpy Philox generator keyed by a 64-bit seed."""
    return np.random.Generator(np.random.Philox(key=int(seed) & _U64))


@dataclass(frozen=True, eq=False)
class SketchMatrix:
    """m x d projection with its seed provenance (read-only entries)."""

    entries: np.ndarray
    seed: int
    orthogonalized: bool = False

    def __post_init__(self) -> None:
        if self.entries.ndim != 2:
            raise ValueError("sketch entries must be a 2-D array")

    @property
    def m(self) -> int:
        return int(self.entries.shape[0])

    @property
    def d(self) -> int:
        return int(self.entries.shape[1])


def _frozen(a: np.ndarray) -> np.ndarray:
    a.setflags(write=False)
    return a


def generate_gaussian(m: int, d: int, seed: int) -> SketchMatrix:
    """i.i.d. N(0, 1) m x d matrix, bit-reproducible in (m, d, seed)."""
    if m < 1 or d < 1:
        raise ValueError(f"sketch dimensions must be positive, got m={m}, d={d}")
    draw = rng_from_seed(seed).standard_normal((m, d))
    return SketchMatrix(entries=_frozen(draw), seed=int(seed), orthogonalized=False)


def orthogonalize(sketch: SketchMatrix) -> SketchMatrix:
    """Row-orthogonalize each block of <= d consecutive rows; rows get norm sqrt(d)."""
    m, d = sketch.m, sketch.d
    rows = []
    for lo in range(0, m, d):
        block = sketch.entries[lo : lo + d]
        q_fac, r_fac = np.linalg.qr(block.T)
        flip = np.sign(np.diagonal(r_fac)).copy()
        flip[flip == 0] = 1.0
        rows.append((q_fac * flip).T)
    out = np.concatenate(rows, axis=0) * np.sqrt(d)
    return SketchMatrix(entries=_frozen(np.ascontiguousarray(out)), seed=sketch.seed,
                        orthogonalized=True)


def round_to_operand(entries: np.ndarray, dtype: str) -> np.ndarray:
    """Round S once to the device operand dtype and return it as float64.

    SURVEY parity decision 1: the device MMA consumes S in bf16 (bf16 / fp32
    keys) or fp16 (fp16 keys); the oracle must receive the *same* rounded S.
    ``dtype`` in {"f64", "f32", "bf16", "f16"}.
    """
    import torch

    t = torch.from_numpy(np.array(entries, dtype=np.float64))
    tdt = {"f64": torch.float64, "f32": torch.float32, "bf16": torch.bfloat16,
           "f16": torch.float16}[dtype]
    return t.to(tdt).to(torch.float64).numpy()
