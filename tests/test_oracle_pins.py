"""Pins of the CPU oracle to what the paper and the mathematics fix.

Each test names the pin and the passage it
comes from.  None of them re-types the oracle's own formula: they compare
against values the paper prints (tests/golden/), closed forms written
differently (the modulo form of PAPER.md:244), brute force over tiny spaces,
exact rational arithmetic, or a library routine (NumPy).
"""
import json
import os
from fractions import Fraction

import numpy as np
import pytest

import oracle
import synth
from tests.exact import exact_fma_f32, round_to_f32

GOLD = os.path.join(os.path.dirname(__file__), "golden")
U64 = 2**64


def gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def h(x):
    return int(x, 16) if isinstance(x, str) else x


# ---------------------------------------------------------------------------
# P1, P2: values the paper prints
# ---------------------------------------------------------------------------

def test_p1_paper_mask_example():
    g = gold("paper_fence_examples.json")["mask_16MiB"]
    base, size = h(g["base"]), g["size"]
    assert oracle.mask(size) == h(g["mask"])
    end_incl = h(g["end_inclusive"])
    # identity at both edges of the partition
    assert oracle.fence_mask(base, base, size) == base
    assert oracle.fence_mask(end_incl, base, size) == end_incl
    # one past the end wraps to the beginning ("start from the beginning")
    assert oracle.fence_mask(end_incl + 1, base, size) == base


def test_p1_small_masks():
    for size, m in gold("paper_fence_examples.json")["mask_small"]["pairs"]:
        assert oracle.mask(size) == h(m)


def test_p2_figure4_wrap():
    g = gold("paper_fence_examples.json")["figure4_wrap"]
    assert oracle.fence_mask(h(g["raw"]), h(g["base"]), g["size"]) == h(g["fenced"])


# ---------------------------------------------------------------------------
# P3, P4, P5, P6: identity, containment, the modulo closed form, AND-then-OR
# ---------------------------------------------------------------------------

def _closed_form(a, base, size, w):
    """base + ((addr - base) % size), rounded down to w."""
    off = ((a.astype(np.uint64) - np.uint64(base)) % np.uint64(size))
    off = (off // np.uint64(w)) * np.uint64(w)
    return np.uint64(base) + off


def test_p5_bruteforce_12bit_space():
    """Every address of a 12-bit space, every pow2 size, every aligned base."""
    a = np.arange(4096, dtype=np.uint64)
    for k in range(0, 13):
        size = 1 << k
        for base in range(0, 4096, size):
            for w in (1, 4, 16):
                if w > size:
                    continue
                got = oracle.fence_mask_n(a, base, size, w)
                np.testing.assert_array_equal(got, _closed_form(a, base, size, w))


def test_p3_p4_p5_toy_arena_all_addresses():
    """All 2^20 addresses of the C1 arena plus 2^20 on each side (P3, P4, P5)."""
    arena = 0x7FA2C0000000
    a = np.arange(arena - (1 << 20), arena + (2 << 20), dtype=np.uint64)
    for t in range(synth.C1_TENANTS):
        base, size = arena + t * synth.C1_PART, synth.C1_PART
        got = oracle.fence_mask_n(a, base, size, 1)
        np.testing.assert_array_equal(got, _closed_form(a, base, size, 1))
        inside = (a >= base) & (a < base + size)
        np.testing.assert_array_equal(got[inside], a[inside])                # P3 identity
        assert ((got >= base) & (got < base + size)).all()                   # P4 containment


def test_p4_p5_random_64bit():
    rng = np.random.Generator(np.random.PCG64(7))
    a = rng.integers(0, U64, 1_000_000, dtype=np.uint64)
    arena = 1 << 40
    for t in (0, 3, 7):
        base, size = arena + t * (1 << 34), 1 << 34
        for w in (1, 4, 16):
            got = oracle.fence_mask_n(a, base, size, w)
            np.testing.assert_array_equal(got, _closed_form(a, base, size, w))
            assert ((got >= base) & (got + np.uint64(w) <= base + size)).all()
            assert (got % np.uint64(w) == 0).all()


def test_p6_and_then_or_has_teeth():
    """OR-then-AND would fail the containment the oracle passes (Listing 1)."""
    base, size = 0x7FA2D0000000, 1 << 24
    a = np.array([0x7FA2CF000010, 0x10, 0xFFFFFFFFFFFFFFF0], dtype=np.uint64)
    wrong = (a | np.uint64(base)) & np.uint64(size - 1)
    assert not ((wrong >= base) & (wrong < base + size)).all()
    got = oracle.fence_mask_n(a, base, size, 1)
    assert ((got >= base) & (got < base + size)).all()


# ---------------------------------------------------------------------------
# P7: the check predicate
# ---------------------------------------------------------------------------

def test_p7_check_bruteforce_byte_membership():
    """ok(a, w) iff every byte a..a+w-1 is in the partition and a % w == 0,
    checked by enumerating bytes over a 12-bit space."""
    a = np.arange(4096, dtype=np.uint64)
    for k in range(4, 13):
        size = 1 << k
        for base in range(0, 4096, size):
            member = np.zeros(4096 + 32, dtype=bool)
            member[base:base + size] = True
            for w in (1, 2, 4, 8, 16):
                every = np.ones(4096, dtype=bool)
                for b in range(w):
                    every &= member[np.arange(4096) + b]
                aligned = np.array([x % w == 0 for x in range(4096)])
                np.testing.assert_array_equal(oracle.check_ok_n(a, base, size, w), every & aligned)


def test_p7_check_edges_and_wraparound():
    base, size = 0x7FA2D0000000, 1 << 24
    end = base + size
    assert oracle.check_ok(base, base, size, 4)
    assert not oracle.check_ok(base - 4, base, size, 4)
    assert not oracle.check_ok(base - 1, base, size, 1)
    assert oracle.check_ok(end - 4, base, size, 4)
    assert not oracle.check_ok(end - 3, base, size, 4)      # misaligned and crosses end
    assert not oracle.check_ok(end, base, size, 1)
    assert oracle.check_ok(end - 1, base, size, 1)
    assert not oracle.check_ok(end - 8, base, size, 16)     # straddles end
    assert not oracle.check_ok(base + 2, base, size, 4)     # misaligned
    assert not oracle.check_ok(U64 - 8, base, size, 16)     # 64-bit wraparound
    # a partition at the very top of the address space
    top = U64 - (1 << 12)
    assert oracle.check_ok(U64 - 16, top, 1 << 12, 16)
    assert not oracle.check_ok(0, top, 1 << 12, 16)


def test_check_range_spec_examples():
    g = gold("paper_fence_examples.json")["check_range"]
    base, size = h(g["base"]), g["size"]
    for addr, length, ok in g["cases"]:
        assert oracle.check_range(base, size, h(addr), length) == ok, (addr, length)


def test_check_range_bruteforce():
    rng = np.random.Generator(np.random.PCG64(3))
    base, size = 4096, 4096
    for _ in range(3000):
        addr = int(rng.integers(0, 3 * 4096))
        length = int(rng.integers(0, 64)) if rng.random() < 0.8 else int(rng.integers(0, 9000))
        if length == 0:
            bf = base <= addr <= base + size
        else:
            bf = all(base <= addr + k < base + size for k in range(length))
        assert oracle.check_range(base, size, addr, length) == bf


# ---------------------------------------------------------------------------
# P9: in-bounds kernels reduce to library routines / exact arithmetic
# ---------------------------------------------------------------------------

PBASE = 0x7FA2C0000000
PSIZE = 1 << 20


def _mem():
    return oracle.Mem(PBASE, PSIZE)


@pytest.mark.parametrize("mode", ["none", "mask", "check"])
def test_p9_copy_is_memcpy(mode):
    rng = synth.rng_for(11)
    m = _mem()
    m.buf[:] = synth.random_bytes(rng, PSIZE)
    n = 16 * 1000 + 7
    src, dst = PBASE + 4096, PBASE + 65536
    expect = m.buf.copy()
    expect[65536:65536 + n] = expect[4096:4096 + n]
    c = oracle.copy(m, PBASE, PSIZE, mode, dst, src, n)
    np.testing.assert_array_equal(m.buf, expect)
    assert c.violations == 0 and c.faults == 0
    assert c.accesses == 2 * (1000 + 7)


def test_copy_crossing_end_mask_wraps_to_start_check_drops():
    """dst's last bytes cross end: mask mode lands them at [base, base+over)
    (Figure 4 wrap), check mode refuses exactly those stores."""
    rng = synth.rng_for(12)
    n = 16 * 64 + 5
    over = 16 * 8 + 5
    dst = PBASE + PSIZE - (n - over)
    src = PBASE + 8192
    for mode in ("mask", "check"):
        m = _mem()
        m.buf[:] = synth.random_bytes(rng, PSIZE)
        before = m.buf.copy()
        c = oracle.copy(m, PBASE, PSIZE, mode, dst, src, n)
        srcb = before[8192:8192 + n]
        np.testing.assert_array_equal(m.buf[PSIZE - (n - over):], srcb[:n - over])
        if mode == "mask":
            np.testing.assert_array_equal(m.buf[:over], srcb[n - over:])
            assert c.violations == 0
        else:
            np.testing.assert_array_equal(m.buf[:over], before[:over])
            # refused stores: the 8 whole 16-byte units and the 5 tail bytes past end
            assert c.violations == 8 + 5


def test_p9_saxpy_single_rounding():
    rng = synth.rng_for(13)
    n = 2003
    x, y = synth.uniform_f32(rng, n), synth.uniform_f32(rng, n)
    a = np.float32(1.5)
    m = _mem()
    m.write(PBASE, x)
    m.write(PBASE + 16384, y)
    c = oracle.saxpy(m, PBASE, PSIZE, "mask", float(a), PBASE, PBASE + 16384, n)
    got = m.view(PBASE + 16384, np.float32, n)
    expect = np.array([exact_fma_f32(a, xi, yi) for xi, yi in zip(x, y)], dtype=np.float32)
    np.testing.assert_array_equal(got.view(np.uint32), expect.view(np.uint32))
    assert c.violations == 0


def test_p9_saxpy_is_not_two_roundings():
    """A cancellation case where fmaf differs from a*x+y rounded twice."""
    a = np.float32(1.0 + 2.0**-12)
    x = np.float32(1.0 + 2.0**-12)
    y = np.float32(-(1.0 + 2.0**-11))
    two = np.float32(np.float32(a * x) + y)
    fused = exact_fma_f32(a, x, y)
    assert two != fused
    m = _mem()
    m.write(PBASE, np.array([x], np.float32))
    m.write(PBASE + 64, np.array([y], np.float32))
    oracle.saxpy(m, PBASE, PSIZE, "none", float(a), PBASE, PBASE + 64, 1)
    assert m.view(PBASE + 64, np.float32, 1)[0] == fused == np.float32(2.0**-24)


@pytest.mark.parametrize("D", [1, 3])
def test_p9_gather_is_take(D):
    rng = synth.rng_for(14)
    T, n = 4096, 1500
    table = synth.uniform_u32(rng, T * D)
    idx = rng.integers(0, T, n).astype(np.int32)
    m = _mem()
    m.write(PBASE, table)
    m.write(PBASE + 4 * T * D, idx)
    out = PBASE + 4 * T * D + 4 * n
    for mode in ("none", "mask", "check"):
        c = oracle.gather(m, PBASE, PSIZE, mode, out, PBASE, PBASE + 4 * T * D, n, D)
        got = m.view(out, np.uint32, n * D)
        np.testing.assert_array_equal(got, table.reshape(T, D)[idx].reshape(-1))
        assert c.violations == 0 and c.accesses == n * (1 + 2 * D)


def test_p9_scatter_add_is_add_at():
    rng = synth.rng_for(15)
    T, n = 512, 5000                                    # many duplicates
    table = synth.uniform_u32(rng, T)
    idx = rng.integers(0, T, n).astype(np.int32)
    src = synth.uniform_u32(rng, n)
    m = _mem()
    m.write(PBASE, table)
    m.write(PBASE + 4096, idx)
    m.write(PBASE + 65536, src)
    expect = table.copy()
    np.add.at(expect, idx, src)                          # uint32, wraps mod 2^32
    c = oracle.scatter_add(m, PBASE, PSIZE, "check", PBASE, PBASE + 4096, PBASE + 65536, n)
    np.testing.assert_array_equal(m.view(PBASE, np.uint32, T), expect)
    assert c.violations == 0


def _stencil_setup(H, W, pitch, field):
    m = _mem()
    inp, out = PBASE, PBASE + 4 * H * pitch
    m.write(inp, field.astype(np.float32).reshape(-1))
    return m, inp, out


def test_p12_stencil_constant_field_exact():
    H, W = 37, 53
    f = np.full((H, W), 0.7123, dtype=np.float32)
    m, inp, out = _stencil_setup(H, W, W, f)
    oracle.stencil(m, PBASE, PSIZE, "mask", out, inp, H, W, W, 0.5, 0.125)
    o = m.view(out, np.float32, H * W).reshape(H, W)
    assert (o[1:-1, 1:-1] == np.float32(0.7123)).all()
    assert (o[0] == 0).all() and (o[-1] == 0).all() and (o[:, 0] == 0).all() and (o[:, -1] == 0).all()


def test_p12_stencil_linear_ramp_exact():
    """A dyadic linear ramp is a fixed point of the Jacobi sweep."""
    H, W, pitch = 33, 40, 48
    r = np.arange(H)[:, None] * 0.25 + np.arange(pitch)[None, :] * 0.5
    m, inp, out = _stencil_setup(H, W, pitch, r)
    oracle.stencil(m, PBASE, PSIZE, "check", out, inp, H, W, pitch, 0.5, 0.125)
    o = m.view(out, np.float32, H * pitch).reshape(H, pitch)
    np.testing.assert_array_equal(o[1:H - 1, 1:W - 1], r[1:H - 1, 1:W - 1].astype(np.float32))


def test_p12_stencil_random_matches_slices_and_exact_fma():
    rng = synth.rng_for(16)
    H, W, pitch = 24, 30, 32
    f = synth.uniform_f32(rng, H * pitch, 0.0, 1.0).reshape(H, pitch)
    m, inp, out = _stencil_setup(H, W, pitch, f)
    c0, c1 = np.float32(0.5), np.float32(0.125)
    oracle.stencil(m, PBASE, PSIZE, "none", out, inp, H, W, pitch, float(c0), float(c1))
    o = m.view(out, np.float32, H * pitch).reshape(H, pitch)
    Cc = f[1:H - 1, 1:W - 1]
    s = (f[0:H - 2, 1:W - 1] + f[2:H, 1:W - 1]) + (f[1:H - 1, 0:W - 2] + f[1:H - 1, 2:W])
    t = c0 * Cc
    expect = np.vectorize(lambda si, ti: exact_fma_f32(c1, si, ti), otypes=[np.float32])(s, t)
    np.testing.assert_array_equal(o[1:H - 1, 1:W - 1].view(np.uint32), expect.view(np.uint32))


# ---------------------------------------------------------------------------
# P11: GEMM exact cases, random against float64 NumPy, descriptor rows
# ---------------------------------------------------------------------------

def _bf16(x):
    return (np.asarray(x, np.float32).view(np.uint32) >> 16).astype(np.uint16)


def _f32(b):
    return (b.astype(np.uint32) << 16).view(np.float32)


def _gemm_mem(A, B, M, N, K):
    m = oracle.Mem(PBASE, 1 << 22)
    pa, pb, pc = PBASE, PBASE + (1 << 20), PBASE + (2 << 20)
    m.write(pa, A)
    m.write(pb, B)
    return m, pa, pb, pc


def test_p11_gemm_identity_gives_B_transpose():
    rng = synth.rng_for(17)
    M = K = 128
    N = 96
    A = _bf16(np.eye(M, K))
    B = synth.bf16_bits_uniform(rng, N * K).reshape(N, K)
    m, pa, pb, pc = _gemm_mem(A, B, M, N, K)
    oracle.gemm(m, PBASE, 1 << 22, "mask", pc, pa, pb, M, N, K, K, K, N)
    C = m.view(pc, np.uint16, M * N).reshape(M, N)
    np.testing.assert_array_equal(_f32(C), _f32(B).T)


def test_p11_gemm_all_ones():
    M, N, K = 64, 48, 256
    A = _bf16(np.ones((M, K)))
    B = _bf16(np.ones((N, K)))
    m, pa, pb, pc = _gemm_mem(A, B, M, N, K)
    oracle.gemm(m, PBASE, 1 << 22, "check", pc, pa, pb, M, N, K, K, K, N)
    C = _f32(m.view(pc, np.uint16, M * N))
    assert (C == K).all()


def test_p11_gemm_random_vs_numpy_float64():
    rng = synth.rng_for(18)
    M, N, K = 70, 90, 200
    A = synth.bf16_bits_uniform(rng, M * K).reshape(M, K)
    B = synth.bf16_bits_uniform(rng, N * K).reshape(N, K)
    m, pa, pb, pc = _gemm_mem(A, B, M, N, K)
    oracle.gemm(m, PBASE, 1 << 22, "none", pc, pa, pb, M, N, K, K, K, N)
    C = _f32(m.view(pc, np.uint16, M * N).reshape(M, N)).astype(np.float64)
    ref = _f32(A).astype(np.float64) @ _f32(B).astype(np.float64).T
    rel = np.linalg.norm(C - ref) / np.linalg.norm(ref)
    assert rel < 4e-3                                            # bf16 output rounding only
    # bf16 rounding of the exact fp32 result: at most half an ulp away
    assert (np.abs(C - ref) <= np.abs(ref) * 2.0**-8 + 1e-30).all()


def test_p11_gemm_operand_orientation_has_teeth():
    """C = A B^T, not A B: on square random inputs the two differ grossly."""
    rng = synth.rng_for(22)
    M = N = K = 48
    A = synth.bf16_bits_uniform(rng, M * K).reshape(M, K)
    B = synth.bf16_bits_uniform(rng, N * K).reshape(N, K)
    m, pa, pb, pc = _gemm_mem(A, B, M, N, K)
    oracle.gemm(m, PBASE, 1 << 22, "mask", pc, pa, pb, M, N, K, K, K, N)
    C = _f32(m.view(pc, np.uint16, M * N).reshape(M, N)).astype(np.float64)
    a64, b64 = _f32(A).astype(np.float64), _f32(B).astype(np.float64)
    good, bad = a64 @ b64.T, a64 @ b64
    assert np.linalg.norm(C - good) / np.linalg.norm(good) < 4e-3
    assert np.linalg.norm(C - bad) / np.linalg.norm(bad) > 0.5


def test_p11_gemm_sampled_rows_match_full():
    rng = synth.rng_for(19)
    M, N, K = 40, 24, 64
    A = synth.bf16_bits_uniform(rng, M * K).reshape(M, K)
    B = synth.bf16_bits_uniform(rng, N * K).reshape(N, K)
    m1, pa, pb, pc = _gemm_mem(A, B, M, N, K)
    oracle.gemm(m1, PBASE, 1 << 22, "mask", pc, pa, pb, M, N, K, K, K, N)
    m2, *_ = _gemm_mem(A, B, M, N, K)
    rows = np.array([0, 7, 39], np.uint32)
    oracle.gemm(m2, PBASE, 1 << 22, "mask", pc, pa, pb, M, N, K, K, K, N, rows=rows)
    full = m1.view(pc, np.uint16, M * N).reshape(M, N)
    part = m2.view(pc, np.uint16, M * N).reshape(M, N)
    np.testing.assert_array_equal(part[rows], full[rows])


def test_desc_rows_bruteforce():
    """Rows a descriptor may touch = the longest prefix of rows whose bytes
    all lie in the partition (enumerated row by row)."""
    base, size = 1 << 20, 1 << 16
    rng = np.random.Generator(np.random.PCG64(5))
    for _ in range(400):
        rowbytes = int(rng.integers(1, 65)) * 16
        stride = rowbytes + int(rng.integers(0, 4)) * 16
        rows = int(rng.integers(1, 200))
        p = base + int(rng.integers(0, size // 16)) * 16
        for mode in ("check", "mask"):
            got, pf = oracle.desc_rows(base, size, mode, p, rows, rowbytes, stride)
            assert pf == p                                  # in-partition start: no move
            bf = 0
            while bf < rows and p + bf * stride + rowbytes <= base + size:
                bf += 1
            assert got == bf
    # start outside the partition: check refuses everything; mask fences the start
    got, _ = oracle.desc_rows(base, size, "check", base - 4096, 10, 64, 64)
    assert got == 0
    got, pf = oracle.desc_rows(base, size, "mask", base - 4096, 10, 64, 64)
    assert pf == base + size - 4096 and got == 10 and oracle.desc_rows(base, size, "none", 7, 10, 64, 64)[0] == 10


def test_p11_gemm_clamped_rows_are_zero_and_counted():
    """A placed so its last rows lie past end: those C rows are exactly 0 and
    check mode counts the refused rows (SURVEY.md §8(d) C4 adversarial part)."""
    rng = synth.rng_for(20)
    M, N, K = 64, 32, 64
    size = 1 << 16
    base = PBASE
    m = oracle.Mem(base, size)
    A = synth.bf16_bits_uniform(rng, M * K).reshape(M, K)
    B = synth.bf16_bits_uniform(rng, N * K).reshape(N, K)
    past = 8
    pa = base + size - (M - past) * K * 2
    pb, pc = base, base + 8192
    m.write(pb, B)
    m.write(pa, A[:M - past])
    for mode in ("mask", "check"):
        c = oracle.gemm(m, base, size, mode, pc, pa, pb, M, N, K, K, K, N)
        C = _f32(m.view(pc, np.uint16, M * N).reshape(M, N))
        assert (C[M - past:] == 0).all()
        ref = _f32(A[:M - past]).astype(np.float64) @ _f32(B).astype(np.float64).T
        assert np.abs(C[:M - past] - ref).max() <= np.abs(ref).max() * 2.0**-7
        assert c.violations == (past if mode == "check" else 0)


# ---------------------------------------------------------------------------
# P8, P10: planted counts and the wrap location on the C1 toy
# ---------------------------------------------------------------------------

ARENA = 0x7FA2C0000000


def _toy_arena(g):
    m = oracle.Mem(ARENA, synth.C1_ARENA)
    for t in range(synth.C1_TENANTS):
        b = ARENA + t * synth.C1_PART
        m.write(b + synth.C1_TABLE_OFF, g.tables[t])
        m.write(b + synth.C1_IDX_OFF, g.idx[t])
    return m


def test_p8_c1_planted_count_and_generator():
    c = gold("c1_toy_counts.json")
    g = synth.toy_gather()
    assert g.n_planted == c["planted_oob"] == synth.planted_count(0.01, c["indices_total"])
    assert sum(int(x.sum()) for x in g.oob_mask) == c["planted_oob"]
    c3 = gold("c3_counts.json")
    for p, k in c3["planted"].items():
        assert synth.planted_count(float(p), c3["indices"]) == k


def test_p8_p2_c1_check_and_mask_modes():
    g = synth.toy_gather()
    total = 0
    for mode in ("check", "mask"):
        m = _toy_arena(g)
        total = 0
        for t in range(synth.C1_TENANTS):
            b = ARENA + t * synth.C1_PART
            before = m.buf.copy()
            c = oracle.gather(m, b, synth.C1_PART, mode, b + synth.C1_OUT_OFF,
                              b + synth.C1_TABLE_OFF, b + synth.C1_IDX_OFF, synth.C1_N, 1)
            assert c.faults == 0
            total += c.violations
            # victims untouched: every byte outside this partition is unchanged
            lo, hi = t * synth.C1_PART, (t + 1) * synth.C1_PART
            np.testing.assert_array_equal(m.buf[:lo], before[:lo])
            np.testing.assert_array_equal(m.buf[hi:], before[hi:])
            out = m.view(b + synth.C1_OUT_OFF, np.uint32, synth.C1_N)
            j = g.idx[t].astype(np.int64)
            inb = ~g.oob_mask[t]
            np.testing.assert_array_equal(out[inb], g.tables[t][j[inb]])
            part_words = before[lo:hi].view(np.uint32)
            if mode == "check":
                assert (out[g.oob_mask[t]] == 0).all()
            else:
                # Figure 4: the wrapped word is word (j mod 65536) of the own partition
                w = np.mod(j[g.oob_mask[t]], 65536)
                np.testing.assert_array_equal(out[g.oob_mask[t]], part_words[w])
        assert total == (655 if mode == "check" else 0)


def test_c1_unfenced_neighbour_reads_victim():
    """Without protection a neighbour index reads another tenant's table
    (the attack of PAPER.md:230 Figure 4); the fence redirects it home."""
    g = synth.toy_gather()
    m = _toy_arena(g)
    arena_words = m.buf.view(np.uint32).copy()
    for t in range(synth.C1_TENANTS):
        b = ARENA + t * synth.C1_PART
        oracle.gather(m, ARENA, synth.C1_ARENA, "none", b + synth.C1_OUT_OFF,
                      b + synth.C1_TABLE_OFF, b + synth.C1_IDX_OFF, synth.C1_N, 1)
        out = m.view(b + synth.C1_OUT_OFF, np.uint32, synth.C1_N)
        nb = g.oob_class[t] == 1
        j = g.idx[t].astype(np.int64)[nb]
        np.testing.assert_array_equal(out[nb], arena_words[t * 65536 + j])
        assert nb.any()


def test_p10_pattern_closed_form_small():
    """Mask-mode gather of j < 0 returns P((size + 4j) mod size) from the
    address-revealing pattern region; check mode returns 0."""
    size = 1 << 20
    base = ARENA
    rng = synth.rng_for(21)
    T, n = 1 << 14, 4096
    pat_lo = 96 * 1024
    m = oracle.Mem(base, size)
    offs = np.arange(pat_lo, size, 4, dtype=np.uint64)
    m.write(base + pat_lo, synth.pattern_words(offs))
    m.write(base, synth.uniform_u32(rng, T))
    j = -rng.integers(1, (size - pat_lo) // 4 + 1, n)
    m.write(base + 65536, j.astype(np.int32))
    out = base + 80 * 1024
    c = oracle.gather(m, base, size, "mask", out, base, base + 65536, n, 1)
    expect = synth.pattern_words(np.mod(size + 4 * j, size).astype(np.uint64))
    np.testing.assert_array_equal(m.view(out, np.uint32, n), expect)
    assert c.violations == 0
    c = oracle.gather(m, base, size, "check", out, base, base + 65536, n, 1)
    assert (m.view(out, np.uint32, n) == 0).all() and c.violations == n


def test_bf16_rounding_pins():
    """RNE to bf16: ties to even, exact values pass through."""
    assert oracle.f32_to_bf16(1.0) == 0x3F80
    assert oracle.f32_to_bf16(1.0 + 2.0**-8) == 0x3F80          # tie -> even (down)
    assert oracle.f32_to_bf16(1.0 + 3 * 2.0**-8) == 0x3F82      # tie -> even (up)
    assert oracle.f32_to_bf16(1.0 + 2.0**-8 + 2.0**-20) == 0x3F81
    assert oracle.bf16_to_f32(0xC000) == -2.0
    rng = np.random.Generator(np.random.PCG64(4))
    for v in rng.uniform(-100, 100, 200).astype(np.float32):
        got = oracle.bf16_to_f32(oracle.f32_to_bf16(float(v)))
        # exact nearest bf16 by rational comparison of the two neighbours
        lo = float(((np.float32(v).view(np.uint32) >> 16) << 16).astype(np.uint32).view(np.float32))
        hi_bits = ((np.float32(v).view(np.uint32) >> 16) + 1) << 16
        hi = float(np.uint32(hi_bits).view(np.float32))
        dl, dh = abs(Fraction(float(v)) - Fraction(lo)), abs(Fraction(float(v)) - Fraction(hi))
        assert got == (lo if dl < dh else hi if dh < dl else got)
    assert round_to_f32(Fraction(1, 3)) == np.float32(1 / 3)
