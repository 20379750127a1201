"""GPU parity of the fenced tcgen05 GEMM against the CPU oracle.

Bar (BASELINE.json north_star): relative Frobenius error <= 1e-2 against the
oracle (fp64 accumulation -> fp32 -> bf16); exact cases (identity, all-ones,
clamped rows) must be bit-exact; every byte outside the stored C rows must
equal the oracle's (nothing else written); check-mode violations exact.
"""
import numpy as np
import pytest

import oracle
import synth
from tests.gpu_util import download, first_diff, upload

pytestmark = pytest.mark.gpu

MiB = 1 << 20
PART = 16 * MiB


def _bf16_to_f32(b):
    return (b.astype(np.uint32) << 16).view(np.float32)


def _setup(arenas, tenants=2):
    a = arenas(tenants * PART)
    parts = [a.partition_alloc(PART) for _ in range(tenants)]
    return a, parts


def _run(a, p, mode, A, B, C, M, N, K, lda, ldb, ldc, exact=False, expect_viol=None):
    before = download(p.base, p.size)
    a.stats_reset()
    a.gemm(p.id, mode, C, A, B, M, N, K, lda, ldb, ldc)
    assert a.device_flags() == 0, "tensor-core pipeline timed out"
    st = a.stats(p.id)
    got = download(p.base, p.size)
    mem = oracle.Mem(p.base, buf=before.copy())
    c = oracle.gemm(mem, p.base, p.size, mode, C, A, B, M, N, K, lda, ldb, ldc)
    assert st["violations"] == c.violations
    if expect_viol is not None:
        assert c.violations == expect_viol
    # region of C that may differ by rounding: stored rows x N columns
    cmask = np.zeros(p.size, bool)
    rows, Cf = oracle.desc_rows(p.base, p.size, mode, C, M, 2 * N, 2 * ldc)
    for i in range(rows):
        o = Cf - p.base + 2 * i * ldc
        cmask[o:o + 2 * N] = True
    assert np.array_equal(got[~cmask], mem.buf[~cmask]), first_diff(got[~cmask], mem.buf[~cmask])
    if rows == 0:
        return c
    g = _bf16_to_f32(got[cmask].view(np.uint16)).astype(np.float64)
    r = _bf16_to_f32(mem.buf[cmask].view(np.uint16)).astype(np.float64)
    if exact:
        np.testing.assert_array_equal(g, r)
    else:
        nr = np.linalg.norm(r)
        rel = np.linalg.norm(g - r) / (nr if nr else 1.0)
        assert rel <= 1e-2, rel
        # element-wise (DESIGN.md R-GEMM): |g - r| <= 2 ulp_bf16(r) + 2^-16 S, S = sum_k |a_k b_k|
        # <= K for the U[-1,1) operands here
        tol = 2 * bf16_ulp(r) + 2.0 ** -16 * K
        bad = np.abs(g - r) > tol
        assert not bad.any(), (int(bad.sum()), float(np.abs(g - r).max()))
        print(f"gemm {M}x{N}x{K} {mode}: rel Frobenius {rel:.2e}, max |err| {np.abs(g - r).max():.2e}")
    return c


def bf16_ulp(x):
    """Spacing of bf16 numbers at |x| (8 significant bits): 2^(e-8) for
    |x| = m 2^e, 0.5 <= m < 1; the smallest normal spacing at 0."""
    _, e = np.frexp(np.abs(x))
    return np.ldexp(1.0, np.maximum(e - 8, -133))


@pytest.mark.parametrize("mode", ["none", "mask", "check"])
@pytest.mark.parametrize("M,N,K", [(128, 256, 64), (256, 512, 256), (200, 304, 128), (384, 768, 1024)])
def test_gemm_random(arenas, mode, M, N, K):
    a, parts = _setup(arenas)
    p = parts[1]
    rng = synth.rng_for(400 + M + N + K)
    A = synth.bf16_bits_uniform(rng, M * K)
    B = synth.bf16_bits_uniform(rng, N * K)
    pa, pb, pc = p.base, p.base + 4 * MiB, p.base + 8 * MiB
    upload(pa, A)
    upload(pb, B)
    _run(a, p, mode, pa, pb, pc, M, N, K, K, K, N, expect_viol=0)


def test_gemm_strided_operands(arenas):
    a, parts = _setup(arenas)
    p = parts[0]
    M, N, K, lda, ldb, ldc = 256, 256, 128, 136, 192, 264
    rng = synth.rng_for(401)
    upload(p.base, synth.bf16_bits_uniform(rng, M * lda))
    upload(p.base + 4 * MiB, synth.bf16_bits_uniform(rng, N * ldb))
    _run(a, p, "mask", p.base, p.base + 4 * MiB, p.base + 8 * MiB, M, N, K, lda, ldb, ldc, expect_viol=0)


def test_gemm_identity_is_exact(arenas):
    a, parts = _setup(arenas)
    p = parts[1]
    M = K = 256
    N = 512
    A = np.zeros((M, K), np.float32)
    np.fill_diagonal(A, 1.0)
    A = (A.view(np.uint32) >> 16).astype(np.uint16)
    B = synth.bf16_bits_uniform(synth.rng_for(402), N * K)
    upload(p.base, A)
    upload(p.base + 4 * MiB, B)
    _run(a, p, "mask", p.base, p.base + 4 * MiB, p.base + 8 * MiB, M, N, K, K, K, N, exact=True)


def test_gemm_all_ones_exact(arenas):
    a, parts = _setup(arenas)
    p = parts[1]
    M, N, K = 128, 256, 512
    one = np.uint16(0x3F80)
    upload(p.base, np.full(M * K, one, np.uint16))
    upload(p.base + 4 * MiB, np.full(N * K, one, np.uint16))
    _run(a, p, "check", p.base, p.base + 4 * MiB, p.base + 8 * MiB, M, N, K, K, K, N, exact=True)
    got = download(p.base + 8 * MiB, 2 * M * N).view(np.uint16)
    assert (_bf16_to_f32(got) == K).all()


@pytest.mark.parametrize("mode", ["mask", "check", "maskcount", "clamp"])
def test_gemm_A_past_end_rows_are_zero(arenas, mode):
    """A placed so its last 64 rows lie past end: the
    descriptor clamp reads them as zero, so those C rows are exactly 0."""
    a, parts = _setup(arenas)
    p = parts[0]
    M, N, K = 256, 256, 256
    rng = synth.rng_for(403)
    pa = p.end - (M - 64) * K * 2
    upload(pa, synth.bf16_bits_uniform(rng, (M - 64) * K))
    upload(p.base, synth.bf16_bits_uniform(rng, N * K))
    pc = p.base + 4 * MiB
    _run(a, p, mode, pa, p.base, pc, M, N, K, K, K, N, expect_viol=0 if mode == "mask" else 64)
    C = download(pc, 2 * M * N).view(np.uint16).reshape(M, N)
    assert (C[M - 64:] == 0).all()


@pytest.mark.parametrize("mode", ["mask", "check", "maskcount", "clamp"])
def test_gemm_C_past_end_rows_not_stored(arenas, mode):
    a, parts = _setup(arenas)
    p = parts[1]
    M, N, K = 256, 512, 128
    rng = synth.rng_for(404)
    upload(p.base, synth.bf16_bits_uniform(rng, M * K))
    upload(p.base + 4 * MiB, synth.bf16_bits_uniform(rng, N * K))
    upload(p.base + 8 * MiB, synth.random_bytes(rng, 8 * MiB))
    pc = p.end - (M - 30) * N * 2                          # last 30 rows of C past end
    _run(a, p, mode, p.base, p.base + 4 * MiB, pc, M, N, K, K, K, N, expect_viol=0 if mode == "mask" else 30)


@pytest.mark.parametrize("mode", ["mask", "check", "maskcount", "clamp"])
def test_gemm_operand_in_victim(arenas, mode):
    """B points into another tenant's partition: check reads no rows (C = 0),
    mask fences the descriptor start into the own partition, clamp moves it
    to the own base (the partition below is the victim)."""
    a, parts = _setup(arenas)
    p, victim = parts[1], parts[0]
    M, N, K = 128, 256, 128
    rng = synth.rng_for(405)
    upload(p.base, synth.bf16_bits_uniform(rng, M * K))
    upload(victim.base + 4 * MiB, synth.bf16_bits_uniform(rng, N * K))
    upload(p.base + 4 * MiB, synth.bf16_bits_uniform(rng, N * K))       # what the mask lands on
    if mode == "clamp":
        assert victim.base < p.base
    vb = download(victim.base, victim.size)
    _run(a, p, mode, p.base, victim.base + 4 * MiB, p.base + 8 * MiB, M, N, K, K, K, N,
         expect_viol=0 if mode == "mask" else N)
    assert np.array_equal(download(victim.base, victim.size), vb)


@pytest.mark.parametrize("seed", range(10))
def test_gemm_fuzz(arenas, seed):
    """Random ragged shapes (M any, N % 16, K % 64), padded strides and, in
    the counting modes, A or C straddling the end or C below the base; both
    1-SM (M < 256) and 2-SM paths."""
    a, parts = _setup(arenas)
    p = parts[seed % 2]
    rng = synth.rng_for(420 + seed)
    mode = ["none", "mask", "check", "modulo", "maskcount", "clamp"][seed % 6]
    M = int(rng.integers(1, 600))
    N = 16 * int(rng.integers(1, 40))
    K = 64 * int(rng.integers(1, 9))
    lda, ldb, ldc = K + 8 * int(rng.integers(0, 4)), K + 8 * int(rng.integers(0, 4)), N + 8 * int(rng.integers(0, 4))
    A, B, C = p.base + 2 * MiB, p.base + 4 * MiB, p.base + 8 * MiB
    if mode in ("check", "maskcount", "clamp"):
        # one operand straddles the end or C lies below the base; operands
        # never overlap (their fenced images stay disjoint too: race-free)
        case = int(rng.integers(0, 3))
        if case == 0:
            A = p.end - 16 * int(rng.integers(1, (M * lda * 2) // 16 + 1))
        elif case == 1:
            C = p.end - 16 * int(rng.integers(1, (M * ldc * 2) // 16 + 1))
        else:
            C = p.base - 16 * int(rng.integers(1, 1 << 12))
    upload(A, synth.bf16_bits_uniform(rng, min(M * lda, (p.end - A) // 2)))
    upload(B, synth.bf16_bits_uniform(rng, N * ldb))
    _run(a, p, mode, A, B, C, M, N, K, lda, ldb, ldc)
