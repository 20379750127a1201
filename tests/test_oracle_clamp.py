"""Pins of the oracle's two counting variants.

* clamp ("compare, clamp and set a violation flag", north_star; the A1
  GD_CHECK_SATURATE variant): an access goes to the largest w-aligned address
  of the partition at or below it, or to the base when there is none; it is
  counted when the check predicate refuses it.
* mask-count (A14 "an optional GD_FLAG_COUNT adds detection"): the access goes
  where the mask fence puts it and is counted when it lies outside the
  partition.

Pinned by enumeration over tiny spaces (the clamp target found by searching
the partition's aligned addresses, the count by byte membership), by the
planted counts of the C1 toy (655, P8), by closed forms of whole kernels
(NumPy: the last refused unit wins an edge slot; `np.add.at` at the clamped
index), and by equality of mask-count data with the independently pinned
mask mode.
"""
import numpy as np
import pytest

import oracle
import synth

U64 = 2**64


def _bytes_inside(a, w, base, size):
    return all(base <= (a + k) < base + size for k in range(w)) and a + w <= U64


def test_clamp_bruteforce_12bit():
    """F(a) = max{x : x w-aligned, [x, x+w) in the partition, x <= a}, else
    base -- found by enumerating the partition, for pow2 and non-pow2 sizes."""
    for size in (16, 48, 64, 208, 1024, 3072):
        for base in (0, 16, 256, 1024 + 48):
            if base % 16:
                continue
            a = np.arange(0, 4096 + 512, dtype=np.uint64)
            for w in (1, 2, 4, 8, 16):
                got = oracle.fence_clamp_n(a, base, size, w)
                cand = np.arange(base, base + size - w + 1, w, dtype=np.int64)
                for ai, gi in zip(a[::3].astype(np.int64), got[::3].astype(np.int64)):
                    below = cand[cand <= ai]
                    want = below[-1] if below.size else base
                    assert gi == want, (size, base, w, ai)


def test_clamp_containment_identity_and_far_addresses():
    rng = np.random.Generator(np.random.PCG64(41))
    a = rng.integers(0, 2**64, 200_000, dtype=np.uint64)
    for size in (1 << 12, 12 << 20, 1 << 34, 3 * (1 << 30)):
        base = (int(rng.integers(1 << 40, 1 << 44)) // size) * size if size & (size - 1) == 0 else \
            int(rng.integers(1 << 40, 1 << 44)) & ~15
        for w in (1, 4, 16):
            f = oracle.fence_clamp_n(a, base, size, w)
            assert ((f >= np.uint64(base)) & (f + np.uint64(w) <= np.uint64(base + size))).all()
            assert ((f - np.uint64(base)) % np.uint64(w) == 0).all()
            lo = a < np.uint64(base)
            hi = a > np.uint64(base + size - w)
            assert (f[lo] == np.uint64(base)).all() and (f[hi] == np.uint64(base + size - w)).all()
        inside = np.arange(base, base + size, max(16, (size // 4099) & ~15), dtype=np.uint64)
        np.testing.assert_array_equal(oracle.fence_clamp_n(inside, base, size, 16), inside)
    # 64-bit extremes
    assert oracle.fence_clamp(0, 1 << 40, 1 << 20, 4) == 1 << 40
    assert oracle.fence_clamp(2**64 - 1, 1 << 40, 1 << 20, 4) == (1 << 40) + (1 << 20) - 4


@pytest.mark.parametrize("mode", ["clamp", "maskcount"])
def test_counted_is_byte_membership_bruteforce(mode):
    """The count of both variants is the check predicate, pinned by byte
    membership (independent of or_check_ok's single-compare form)."""
    base, size = 512, 256
    m = oracle.Mem(0, 8)
    c = m.ctx(base, size, mode)
    for w in (1, 4, 16):
        for a in range(0, 1024):
            want = not (_bytes_inside(a, w, base, size) and a % w == 0)
            assert bool(oracle.lib().or_counted(c, a, w)) == want, (w, a)
        for a in (U64 - 16, U64 - 1, 2**63):
            assert oracle.lib().or_counted(c, a, w) == 1


def test_maskcount_resolves_like_mask_12bit():
    a = np.arange(4096, dtype=np.int64)
    for k in (4, 8, 10):
        size = 1 << k
        for base in range(0, 4096, size * 3):
            for w in (1, 4, 16):
                want = oracle.fence_mask_n(a.astype(np.uint64), base, size, w)
                got = [oracle.resolve(base, size, "maskcount", int(x), w) for x in a[::17]]
                assert all(ok for _, ok in got)
                assert [r for r, _ in got] == [int(v) for v in want[::17]]


# ---------------------------------------------------------------------------
# whole kernels
# ---------------------------------------------------------------------------

ARENA = 0x7FA2C0000000


def _toy_arena(g):
    m = oracle.Mem(ARENA, synth.C1_ARENA)
    for t in range(synth.C1_TENANTS):
        b = ARENA + t * synth.C1_PART
        m.write(b + synth.C1_TABLE_OFF, g.tables[t])
        m.write(b + synth.C1_IDX_OFF, g.idx[t])
    return m


def test_c1_toy_maskcount_and_clamp():
    """C1: both variants count exactly the 655 planted indices (P8).
    mask-count outputs equal mask mode's; clamp outputs read the partition's
    first word (targets below the base) or last word (above the end)."""
    g = synth.toy_gather()
    outs = {}
    for mode in ("mask", "maskcount", "clamp"):
        m = _toy_arena(g)
        total = 0
        outs[mode] = []
        for t in range(synth.C1_TENANTS):
            b = ARENA + t * synth.C1_PART
            before = m.buf.copy()
            c = oracle.gather(m, b, synth.C1_PART, mode, b + synth.C1_OUT_OFF,
                              b + synth.C1_TABLE_OFF, b + synth.C1_IDX_OFF, synth.C1_N, 1)
            assert c.faults == 0
            total += c.violations
            lo, hi = t * synth.C1_PART, (t + 1) * synth.C1_PART
            np.testing.assert_array_equal(m.buf[:lo], before[:lo])
            np.testing.assert_array_equal(m.buf[hi:], before[hi:])
            out = m.view(b + synth.C1_OUT_OFF, np.uint32, synth.C1_N).copy()
            outs[mode].append(out)
            j = g.idx[t].astype(np.int64)
            inb = ~g.oob_mask[t]
            np.testing.assert_array_equal(out[inb], g.tables[t][j[inb]])
            if mode == "clamp":
                part_words = before[lo:hi].view(np.uint32)
                raw = (b + synth.C1_TABLE_OFF) + 4 * j[g.oob_mask[t]]
                want = np.where(raw < b, part_words[0], part_words[-1])
                np.testing.assert_array_equal(out[g.oob_mask[t]], want)
        assert total == (0 if mode == "mask" else 655)
    for a, b_ in zip(outs["mask"], outs["maskcount"]):
        np.testing.assert_array_equal(a, b_)


def test_clamp_copy_crossing_end_last_unit_wins():
    """dst's last units lie past end: in clamp mode each goes to the last
    16 bytes of the partition, in ascending order, so the last one wins;
    each refused unit counts once (load or store)."""
    base, size = 1 << 20, 1 << 16
    m = oracle.Mem(base, size)
    rng = synth.rng_for(51)
    src = base
    n, over = 4096 + 48, 96                       # 6 units past end
    data = synth.random_bytes(rng, n)
    m.write(src, data)
    dst = base + size - (n - over)
    c = oracle.copy(m, base, size, "clamp", dst, src, n)
    got = m.view(base + size - (n - over), np.uint8, n - over)
    want = data[: n - over].copy()
    want[-16:] = data[n - 16:]                     # the last refused unit's bytes
    np.testing.assert_array_equal(got, want)
    assert c.violations == over // 16


def test_clamp_scatter_add_lands_on_edges():
    """RMWs past either end accumulate at the first / last word (np.add.at at
    the clamped index); counted once each.  Addresses are u64: a negative
    index that wraps below 0 is a huge address, above the partition."""
    base, size = 1 << 24, 1 << 16
    words = size // 4
    rng = synth.rng_for(52)
    n = 3000
    j = rng.integers(0, words // 2, n).astype(np.int64)
    pos = synth.planted_positions(rng, n, 90)
    j[pos[:45]] = rng.integers(-(1 << 30), -1, 45)
    j[pos[45:]] = rng.integers(words // 2 + 1, 1 << 30, 45)   # table at the partition middle
    tab = base + size // 2
    src = rng.integers(0, 2**32, n, dtype=np.uint64).astype(np.uint32)
    m = oracle.Mem(base, size)
    init = rng.integers(0, 2**32, words, dtype=np.uint64).astype(np.uint32)
    init[:32] = 0                                  # idx / src live elsewhere (below)
    m.write(base, init)
    idx_at, src_at = base + 4 * 64, base + 4 * 64 + 4 * n
    assert src_at + 4 * n <= tab
    m.write(idx_at, j.astype(np.int32))
    m.write(src_at, src)
    before = m.view(base, np.uint32, words).copy()
    c = oracle.scatter_add(m, base, size, "clamp", tab, idx_at, src_at, n)
    raw = [(tab + 4 * int(x)) % 2**64 for x in j]          # u64 addresses (A4 sext, mod 2^64)
    k = np.array([0 if r < base else words - 1 if r > base + size - 4 else (r - base) // 4 for r in raw])
    want = before.astype(np.uint64)
    np.add.at(want, k, src.astype(np.uint64))
    np.testing.assert_array_equal(m.view(base, np.uint32, words), (want % 2**32).astype(np.uint32))
    assert c.violations == 90


def test_clamp_desc_rows_and_gemm_count():
    """Descriptor rule in clamp mode: an operand starting below the base is
    moved to the base (rows then counted from there); the count is the check
    count (rows not wholly inside at the unfenced address)."""
    base, size = 1 << 20, 1 << 16
    got, pf = oracle.desc_rows(base, size, "clamp", base - 4096, 10, 64, 64)
    assert pf == base and got == 10
    got, pf = oracle.desc_rows(base, size, "clamp", base + size + 4096, 10, 64, 64)
    assert pf == base + size - 16 and got == 0
    got, pf = oracle.desc_rows(base, size, "clamp", base + size - 5 * 64, 10, 64, 64)
    assert pf == base + size - 5 * 64 and got == 5
    # GEMM: A's last rows past end -> C rows 0; count = refused rows in every counting mode
    M, N, K = 32, 16, 32
    m = oracle.Mem(base, size)
    rng = synth.rng_for(53)
    A = synth.bf16_bits_uniform(rng, M * K).reshape(M, K)
    B = synth.bf16_bits_uniform(rng, N * K).reshape(N, K)
    past = 4
    pa = base + size - (M - past) * K * 2
    m.write(base, B)
    m.write(pa, A[:M - past])
    for mode in ("check", "maskcount", "clamp"):
        c = oracle.gemm(m, base, size, mode, base + 8192, pa, base, M, N, K, K, K, N)
        assert c.violations == past, mode
