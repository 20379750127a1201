"""Pins of the oracle's modulo fence (§4.4).

fenced = base + ((a - base) % size), 64-bit unsigned remainder (reading A10),
rounded down to the access width (A3).  Pinned by
  * equality with the mask fence on power-of-two, size-aligned partitions
    (the paper's two fencing methods agree there; an independent function),
  * a brute-force characterisation for a >= base: the unique address of the
    partition congruent to a modulo size (enumerated, not computed),
  * containment for every address, and the A10 wraparound example.
"""
import numpy as np

import oracle


def test_modulo_equals_mask_on_pow2_bruteforce_12bit():
    a = np.arange(4096, dtype=np.uint64)
    for k in range(4, 13):
        size = 1 << k
        for base in range(0, 4096, size):
            for w in (1, 4, 16):
                np.testing.assert_array_equal(oracle.fence_modulo_n(a, base, size, w),
                                              oracle.fence_mask_n(a, base, size, w))


def test_modulo_congruence_bruteforce_non_pow2():
    """For a >= base: F(a) is the partition address congruent to a mod size
    (found by enumerating the partition), rounded down to w."""
    for size in (48, 80, 96, 208, 1040, 3072):
        for base in (0, 16, 112, 4096 + 48):
            cand = np.arange(base, base + size, dtype=np.int64)
            a = np.arange(base, base + 5 * size + 37, dtype=np.uint64)
            for w in (1, 4, 16):
                got = oracle.fence_modulo_n(a, base, size, w).astype(np.int64)
                for ai, gi in zip(a[::7].astype(np.int64), got[::7]):
                    hit = cand[(cand - ai) % size == 0][0]
                    assert gi == hit - (hit - base) % w, (size, base, w, ai)


def test_modulo_containment_and_identity_random():
    rng = np.random.Generator(np.random.PCG64(31))
    a = rng.integers(0, 2**64, 200_000, dtype=np.uint64)
    for size in (12 << 20, (14 << 20) + 4096, 3 * (1 << 30), 1 << 34):
        base = int(rng.integers(1 << 40, 1 << 44)) & ~15
        for w in (1, 4, 16):
            f = oracle.fence_modulo_n(a, base, size, w)
            assert ((f >= np.uint64(base)) & (f + np.uint64(w) <= np.uint64(base + size))).all()
            assert ((f - np.uint64(base)) % np.uint64(w) == 0).all()
        inside = np.arange(base, base + size, max(1, size // 4099), dtype=np.uint64)
        np.testing.assert_array_equal(oracle.fence_modulo_n(inside, base, size, 1), inside)


def test_modulo_below_base_uses_u64_remainder():
    """Reading A10: for a < base the u64 difference wraps, so a non-pow2 size
    gives (2^64 - d) mod size, not the Euclidean residue (SURVEY.md §8(c) A10:
    offset -5 with size 12288 -> 4091, Euclidean would be 12283)."""
    base, size = 1 << 40, 12288
    assert oracle.fence_modulo(base - 5, base, size, 1) == base + 4091
    assert (2**64 - 5) % 12288 == 4091 and (-5) % 12288 == 12283
    # and for a pow2 size the two readings coincide with the mask fence
    assert oracle.fence_modulo(base - 5, base, 4096, 1) == oracle.fence_mask(base - 5, base, 4096, 1)


def test_modulo_mode_in_simulated_kernel():
    """A copy whose destination crosses end wraps to the partition start in
    modulo mode exactly as the congruence says, for a non-pow2 partition."""
    base, size = 0x7F0000000000, 3 * (1 << 20)
    m = oracle.Mem(base, size)
    rng = np.random.Generator(np.random.PCG64(32))
    m.buf[:] = rng.integers(0, 256, size, dtype=np.uint8)
    n, over = (1 << 20) + 5, 4096 + 5            # dst stays 16-byte aligned
    src = bytes(m.buf[:n])
    dst = base + size - (n - over)
    before = m.buf.copy()
    c = oracle.copy(m, base, size, "modulo", dst, base, n)
    assert c.violations == 0 and c.faults == 0
    np.testing.assert_array_equal(m.buf[size - (n - over):], np.frombuffer(src, np.uint8)[:n - over])
    np.testing.assert_array_equal(m.buf[:over], np.frombuffer(src, np.uint8)[n - over:])
    np.testing.assert_array_equal(m.buf[over:size - (n - over)], before[over:size - (n - over)])
