"""Seeded synthetic input generators shared by the oracle tests and the GPU path.

This module holds NO arithmetic of the method (no fence, no check, no kernel
math): it only draws inputs -- random bytes, floats, indices, and the
positions and values of planted out-of-partition indices -- from NumPy's
PCG64 with the seeds DESIGN.md states (``1000 * config + tenant``).  Both the
oracle tests and the CUDA parity tests take their inputs from here, so the two
sides see identical inputs while sharing no code.

Layouts follow SURVEY.md §8(d) (config table) and reading A8/A9.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

KiB, MiB, GiB = 1 << 10, 1 << 20, 1 << 30

# ---------------------------------------------------------------------------
# C1 toy: 1 MiB arena, 4 tenants x 256 KiB, int32 gather of 4 x 16,384
# indices with 1 % planted out-of-partition indices (BASELINE.json configs[0],
# SURVEY.md reading A8).
# ---------------------------------------------------------------------------
C1_ARENA = 1 * MiB
C1_TENANTS = 4
C1_PART = 256 * KiB
C1_TABLE_OFF, C1_TABLE_N = 0, 32768            # 128 KiB of u32
C1_IDX_OFF, C1_N = 128 * KiB, 16384            # 64 KiB of int32
C1_OUT_OFF = 192 * KiB                         # 64 KiB of u32
C1_OOB_FRAC = 0.01
PATTERN_XOR = 0x9E3779B9


def seed_for(config: int, tenant: int) -> int:
    return 1000 * config + tenant


def planted_count(frac: float, n: int) -> int:
    """k = round_half_even(frac * n) (reading A9)."""
    return int(np.round(frac * n))


def planted_positions(rng: np.random.Generator, n: int, k: int) -> np.ndarray:
    """k distinct positions of [0, n) by a seeded Fisher-Yates shuffle."""
    return np.sort(rng.permutation(n)[:k]).astype(np.int64)


@dataclass
class ToyGather:
    tables: list          # per tenant: uint32[32768]
    idx: list             # per tenant: int32[16384]
    oob_mask: list        # per tenant: bool[16384] True where planted OOB
    oob_class: list       # per tenant: int8[16384]: 0 in-bounds, 1 neighbour, 2 far-neg, 3 far-pos
    n_planted: int


def toy_gather(seed: int = 1000, frac: float = C1_OOB_FRAC) -> ToyGather:
    """C1 inputs.  Planted classes cycle neighbour, far-neg, far-pos over the
    planted positions in ascending order (a third each, every tenant gets all):

    neighbour: j = i' + k*65536, k != 0, raw address in tenant (t+k)'s table;
    far-neg:   j = -m*65536 + r, m in [1, 32767], r in [0, 49152);
    far-pos:   j =  m*65536 + r, m in [1, 32767], r in [0, 49152).
    65536 words = one 256 KiB partition, so each class lies outside the own
    partition, and the low 18 address bits (r or i') keep the wrapped target
    inside [table, idx) -- never in ``out`` (race-free).
    """
    rng = np.random.Generator(np.random.PCG64(seed))
    total = C1_TENANTS * C1_N
    k = planted_count(frac, total)
    pos = planted_positions(rng, total, k)
    classes = np.zeros(total, dtype=np.int8)
    classes[pos] = 1 + (np.arange(k) % 3)
    tables, idxs, masks, clss = [], [], [], []
    for t in range(C1_TENANTS):
        tables.append(rng.integers(0, 2**32, C1_TABLE_N, dtype=np.uint64).astype(np.uint32))
        j = rng.integers(0, C1_TABLE_N, C1_N, dtype=np.int64)
        c = classes[t * C1_N:(t + 1) * C1_N]
        for i in np.nonzero(c)[0]:
            if c[i] == 1:
                ks = [kk for kk in range(-t, C1_TENANTS - t) if kk != 0]
                kk = ks[int(rng.integers(0, len(ks)))]
                j[i] = int(rng.integers(0, C1_TABLE_N)) + kk * 65536
            elif c[i] == 2:
                j[i] = -int(rng.integers(1, 32768)) * 65536 + int(rng.integers(0, 49152))
            else:
                j[i] = int(rng.integers(1, 32768)) * 65536 + int(rng.integers(0, 49152))
        idxs.append(j.astype(np.int32))
        masks.append(c != 0)
        clss.append(c.copy())
    return ToyGather(tables, idxs, masks, clss, k)


def chaos_indices(rng: np.random.Generator, n: int) -> np.ndarray:
    """Any int32, with the extremes forced in (SURVEY.md §8(d) C1 chaos suite)."""
    j = rng.integers(-2**31, 2**31, n, dtype=np.int64)
    extremes = np.array([2**31 - 1, -1, -2**31, 0, 1, -2], dtype=np.int64)
    j[:min(n, extremes.size)] = extremes[:min(n, extremes.size)]
    return j.astype(np.int32)


# ---------------------------------------------------------------------------
# Generic seeded draws
# ---------------------------------------------------------------------------

def rng_for(seed: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(seed))


def random_bytes(rng, n: int) -> np.ndarray:
    return rng.integers(0, 256, n, dtype=np.uint8)


def uniform_f32(rng, n: int, lo=-1.0, hi=1.0) -> np.ndarray:
    return rng.uniform(lo, hi, n).astype(np.float32)


def uniform_u32(rng, n: int) -> np.ndarray:
    return rng.integers(0, 2**32, n, dtype=np.uint64).astype(np.uint32)


def indices_with_oob(rng, n: int, table_n: int, frac: float):
    """Embedding-style indices (C3): in-bounds j uniform in [0, table_n);
    exactly round(frac*n) planted positions with j uniform in [-2^31, 0)
    (raw address below the partition base).  Returns (idx int32, positions)."""
    j = rng.integers(0, table_n, n, dtype=np.int64)
    k = planted_count(frac, n)
    pos = planted_positions(rng, n, k) if k else np.zeros(0, dtype=np.int64)
    if k:
        j[pos] = rng.integers(-2**31, 0, k, dtype=np.int64)
    return j.astype(np.int32), pos


def pattern_words(offsets_bytes: np.ndarray) -> np.ndarray:
    """Address-revealing fill P(o) = (o >> 2) ^ 0x9E3779B9 for byte offset o
    (a word-sized label of its own location)."""
    o = np.asarray(offsets_bytes, dtype=np.uint64)
    return ((o >> np.uint64(2)) ^ np.uint64(PATTERN_XOR)).astype(np.uint32)


def bf16_bits_uniform(rng, n: int, lo=-1.0, hi=1.0) -> np.ndarray:
    """bf16(U[lo,hi)) as raw uint16 bits, by truncating fp32 draws to their
    top 16 bits (an input distribution, not the method's rounding)."""
    f = rng.uniform(lo, hi, n).astype(np.float32)
    return (f.view(np.uint32) >> np.uint32(16)).astype(np.uint16)


def oob_indices(rng, k: int, part_words: int, lo_word: int, hi_word: int, table_word: int = 0,
                below: bool = True) -> np.ndarray:
    """k int32 indices j, relative to a table starting ``table_word`` words
    after the partition base, whose raw word offset ``table_word + j`` lies
    OUTSIDE [0, part_words) (another partition, or outside the arena) while
    its residue mod part_words lies in [lo_word, hi_word) -- so a wrapped
    access lands in a region the test keeps free of same-launch writes
    (race-free).  Half below the base, half above
    (below=False: all above, e.g. for non-power-of-two partitions)."""
    w = rng.integers(lo_word, hi_word, k, dtype=np.int64) - table_word      # residue, relative to table
    below_mask = rng.random(k) < 0.5
    below = below_mask & below
    m_neg = (w + 2**31) // part_words          # largest m with w - m*P >= -2^31
    m_pos = (2**31 - 1 - w) // part_words      # largest m with w + m*P <= 2^31 - 1
    u = rng.random(k)
    j = np.where(below,
                 w - (1 + np.floor(u * np.maximum(m_neg, 1)).astype(np.int64)) * part_words,
                 w + (1 + np.floor(u * np.maximum(m_pos, 1)).astype(np.int64)) * part_words)
    raw = j + table_word
    assert ((raw < 0) | (raw >= part_words)).all()
    assert (j >= -2**31).all() and (j < 2**31).all()
    return j.astype(np.int32)
