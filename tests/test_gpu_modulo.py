"""GPU parity of modulo fencing (§4.4)
on exact-size (non-power-of-two) partitions, against the CPU oracle.

The device computes the 64-bit modulo inline from the reciprocal parameter
floor(2^64/size); the oracle uses the plain u64 remainder.  Layouts keep every
wrapped access race-free; out-of-partition indices lie above the base so the
residue is the plain one (reading A10 covers a < base, tested separately)."""
import numpy as np
import pytest

import oracle
import synth
from paper_2401_09290_b200 import guardian as g
from tests.gpu_util import download, first_diff, upload

pytestmark = pytest.mark.gpu

MiB = 1 << 20
EXACT = 14 * MiB                      # 7 VMM granules: not a power of two


def _setup(arenas, seed):
    a = arenas(64 * MiB)
    parts = [a.partition_alloc_exact(EXACT) for _ in range(3)]
    for p in parts:
        assert p.size == EXACT and not p.pow2
    rng = synth.rng_for(seed)
    for p in parts:
        upload(p.base, synth.random_bytes(rng, p.size))
    return a, parts, rng


def _run(a, parts, t, mode, launch, oracle_fn, expect_violations=None):
    p = parts[t]
    snap = {q.id: download(q.base, q.size) for q in parts}
    a.stats_reset()
    launch(p)
    st = a.stats(p.id)
    mem = oracle.Mem(p.base, buf=snap[p.id].copy())
    c = oracle_fn(mem, p)
    got = download(p.base, p.size)
    assert np.array_equal(got, mem.buf), f"{mode}: {first_diff(got, mem.buf)}"
    for q in parts:
        if q.id != p.id:
            assert np.array_equal(download(q.base, q.size), snap[q.id]), "victim modified"
    assert c.faults == 0 and st["violations"] == c.violations
    if expect_violations is not None:
        assert c.violations == expect_violations


def test_exact_partitions_layout(arenas):
    a = arenas(64 * MiB)
    ps = [a.partition_alloc_exact(EXACT) for _ in range(3)]
    for x, y in zip(ps, ps[1:]):
        assert x.end <= y.base or y.end <= x.base
    with pytest.raises(g.GuardianError) as e:
        a.copy(ps[0].id, "mask", ps[0].base, ps[0].base + 16, 64)
    assert e.value.status == g.GD_ERR_NOT_POW2
    a.partition_free(ps[1].id)
    q = a.partition_alloc(16 * MiB)                 # the freed block and its tail coalesced
    assert q.base % q.size == 0


@pytest.mark.parametrize("mode", ["modulo", "check", "none"])
def test_modulo_copy_crossing_end(arenas, mode):
    a, parts, _ = _setup(arenas, 601)
    n = 3 * MiB + 16 * 9 + 5
    p = parts[1]
    if mode == "none":                                            # in bounds, ending 11 bytes before end
        dst = p.end - (n + 11)
    else:                                                         # the last 512 KiB + 5 bytes cross end
        dst = p.end - (n - (512 * 1024 + 5))
    _run(a, parts, 1, mode,
         lambda p: a.copy(p.id, mode, dst, p.base + 4 * MiB, n),
         lambda m, p: oracle.copy(m, p.base, p.size, mode, dst, p.base + 4 * MiB, n))


@pytest.mark.parametrize("mode", ["modulo", "check"])
def test_modulo_saxpy_crossing_end(arenas, mode):
    a, parts, rng = _setup(arenas, 602)
    n, over = (1 << 19) + 3, (1 << 15) + 3
    p = parts[0]
    upload(p.base + 4 * MiB, synth.uniform_f32(rng, n))
    y = p.end - 4 * (n - over)
    upload(y, synth.uniform_f32(rng, n - over))
    upload(p.base, synth.uniform_f32(rng, over))
    _run(a, parts, 0, mode,
         lambda p: a.saxpy(p.id, mode, 0.625, p.base + 4 * MiB, y, n),
         lambda m, p: oracle.saxpy(m, p.base, p.size, mode, 0.625, p.base + 4 * MiB, y, n),
         None if mode == "modulo" else 2 * over)


@pytest.mark.parametrize("mode", ["modulo", "check"])
def test_modulo_gather_scatter_adversarial(arenas, mode):
    a, parts, rng = _setup(arenas, 603)
    p = parts[2]
    T, n = 1 << 20, (1 << 17) + 3
    j = rng.integers(0, T, n, dtype=np.int64).astype(np.int32)
    k = synth.planted_count(0.02, n)
    pos = synth.planted_positions(rng, n, k)
    j[pos] = synth.oob_indices(rng, k, EXACT // 4, (10 * MiB) // 4, EXACT // 4, below=False)
    upload(p.base + 4 * MiB, j)
    _run(a, parts, 2, mode,
         lambda p: a.gather(p.id, mode, p.base + 6 * MiB, p.base, p.base + 4 * MiB, n),
         lambda m, p: oracle.gather(m, p.base, p.size, mode, p.base + 6 * MiB, p.base, p.base + 4 * MiB, n),
         None if mode == "modulo" else k)
    _run(a, parts, 2, mode,
         lambda p: a.scatter(p.id, mode, p.base, p.base + 4 * MiB, p.base + 6 * MiB, n),
         lambda m, p: oracle.scatter_add(m, p.base, p.size, mode, p.base, p.base + 4 * MiB, p.base + 6 * MiB, n),
         None if mode == "modulo" else k)


@pytest.mark.parametrize("mode", ["modulo", "check"])
def test_modulo_stencil_out_crossing_end(arenas, mode):
    a, parts, rng = _setup(arenas, 604)
    H, W, pitch = 160, 1000, 1024
    p = parts[1]
    upload(p.base + 4 * MiB, synth.uniform_f32(rng, H * pitch, 0.0, 1.0))
    out = p.end - (H - 7) * pitch * 4
    _run(a, parts, 1, mode,
         lambda p: a.stencil(p.id, mode, out, p.base + 4 * MiB, H, W, pitch, 0.5, 0.125),
         lambda m, p: oracle.stencil(m, p.base, p.size, mode, out, p.base + 4 * MiB, H, W, pitch, 0.5, 0.125),
         None if mode == "modulo" else 6 * (W - 2))


@pytest.mark.parametrize("mode", ["modulo", "check"])
@pytest.mark.parametrize("D", [6, 12, 32, 64])       # D = 6: flat words; row slots: tpr 3 (reciprocal), 8 (shift); G = 1, 1, 2
@pytest.mark.parametrize("case", ["out_crossing_end", "idx_below_base"])
def test_modulo_gather_rows_stream_walk(arenas, mode, D, case):
    """Per access (run again by test_gpu_peraccess.py), the row gather fences
    its index and output streams by a walk (Fence::step_up) when a thread's
    ranges neither straddle the base nor span the partition, else by the full
    modulo.  Both paths against the oracle's u64 remainder: `out` running past
    the end of a non-power-of-two partition, and `idx` starting below the base
    (its wrapped half holds valid indices, so every read is race-free)."""
    a, parts, rng = _setup(arenas, 606)
    p = parts[1]
    n = 2048
    tab = p.base + 1 * MiB
    j = rng.integers(0, n, n, dtype=np.int64).astype(np.int32)
    if case == "out_crossing_end":
        idx, out = p.base + 3 * MiB, p.end - n * 4 * D // 2
        upload(idx, j)
    else:
        idx, out = p.base - 4 * (n // 2), p.base + 6 * MiB
        upload(p.base, j[n // 2:])
        # the first half lies below the base: element e is read (modulo) at
        # base + ((idx + 4e - base) mod 2^64) mod size
        for e in range(n // 2):
            upload(p.base + ((idx + 4 * e - p.base) % (1 << 64)) % p.size, j[e:e + 1])
    _run(a, parts, 1, mode,
         lambda p: a.gather(p.id, mode, out, tab, idx, n, D),
         lambda m, p: oracle.gather(m, p.base, p.size, mode, out, tab, idx, n, D))


@pytest.mark.parametrize("mode", ["modulo", "check", "clamp"])
@pytest.mark.parametrize("case", ["in_crossing_end", "in_below_base", "pitch_past_size"])
def test_modulo_stencil_walk(arenas, mode, case):
    """The per-access stencil's modulo fence follows each row's vector from
    the row before (Fence::step_up), the W / E words from the row below
    (step_down) and each output row from the one before, when the strip does
    not straddle the base and a row step is below the partition size; other
    strips take the full modulo per access.  Every path against the oracle's
    plain u64 remainder: the walk stepping over the partition end
    (conditional subtract), `in` starting below the base (strips wholly
    below it walk on wrapped offsets, the straddling strip takes the full
    modulo), and a row step of more than the partition size (full modulo).
    Run hoisted here and per access by test_gpu_peraccess.py."""
    a, parts, rng = _setup(arenas, 605)
    p = parts[1]
    # finite values everywhere a wrapped row can land (random bytes hold NaNs,
    # whose payloads the GPU and the host propagate differently)
    upload(p.base, synth.uniform_f32(rng, p.size // 4, 0.0, 1.0))
    if case == "pitch_past_size":
        if mode == "clamp":
            pytest.skip("the output row lies past the end: its clamped stores collide (reading R-race)")
        H, W, pitch = 3, 200, EXACT // 4 + 4096
        inp = p.base + 4 * MiB
    else:
        H, W, pitch = 160, 1000, 1024
        inp = p.end - 40 * pitch * 4 if case == "in_crossing_end" else p.base - 40 * pitch * 4 - 64
    out = p.base + 1 * MiB
    _run(a, parts, 1, mode,
         lambda p: a.stencil(p.id, mode, out, inp, H, W, pitch, 0.5, 0.125),
         lambda m, p: oracle.stencil(m, p.base, p.size, mode, out, inp, H, W, pitch, 0.5, 0.125))


@pytest.mark.parametrize("mode", ["modulo", "check", "clamp"])
def test_exact_partition_stencil_tma(arenas, mode):
    """K5 v2 on an exact-size (non-power-of-two) partition: `in` far past the
    end (modulo wraps the descriptor base, clamp moves it to the last legal
    16-byte address, check refuses it) and `out` crossing the end."""
    a, parts, rng = _setup(arenas, 607)
    H, W, pitch = 120, 1001, 1004
    p = parts[1]
    inp = p.base + EXACT + 3 * MiB + 64                 # outside, 16-aligned
    upload(p.base + 3 * MiB, synth.uniform_f32(rng, H * pitch, 0.0, 1.0))      # where modulo lands
    upload(p.end - 4 * MiB, synth.uniform_f32(rng, MiB, 0.0, 1.0))
    out = p.end - 60 * 4 * pitch - 4 * (W - 1)
    _run(a, parts, 1, mode,
         lambda p: a.stencil_tma(p.id, mode, out, inp, H, W, pitch, 0.5, 0.125),
         lambda m, p: oracle.stencil_tma(m, p.base, p.size, mode, out, inp, H, W, pitch, 0.5, 0.125),
         None if mode == "modulo" else H + (H - 1 - 61))


@pytest.mark.parametrize("mode", ["modulo", "check"])
def test_modulo_gemm_A_past_end(arenas, mode):
    a, parts, rng = _setup(arenas, 605)
    p = parts[0]
    M, N, K = 256, 256, 128
    pa = p.end - (M - 32) * K * 2
    upload(pa, synth.bf16_bits_uniform(rng, (M - 32) * K))
    upload(p.base, synth.bf16_bits_uniform(rng, N * K))
    pc = p.base + 2 * MiB
    before = download(p.base, p.size)
    a.stats_reset()
    a.gemm(p.id, mode, pc, pa, p.base, M, N, K, K, K, N)
    assert a.device_flags() == 0
    got = download(p.base, p.size)
    mem = oracle.Mem(p.base, buf=before)
    c = oracle.gemm(mem, p.base, p.size, mode, pc, pa, p.base, M, N, K, K, K, N)
    assert a.stats(p.id)["violations"] == c.violations == (32 if mode == "check" else 0)
    cm = np.zeros(p.size, bool)
    cm[2 * MiB:2 * MiB + 2 * M * N] = True
    assert np.array_equal(got[~cm], mem.buf[~cm])
    gg = (got[cm].view(np.uint16).astype(np.uint32) << 16).view(np.float32).astype(np.float64)
    rr = (mem.buf[cm].view(np.uint16).astype(np.uint32) << 16).view(np.float32).astype(np.float64)
    assert np.linalg.norm(gg - rr) / np.linalg.norm(rr) <= 1e-2
    assert (got[cm].view(np.uint16).reshape(M, N)[M - 32:] == 0).all()


def test_modulo_equals_mask_on_pow2_partition(arenas):
    """On a power-of-two partition the two fencing methods are the same
    function: identical results for adversarial indices (incl. j < 0)."""
    a = arenas(64 * MiB)
    p = a.partition_alloc(16 * MiB)
    rng = synth.rng_for(606)
    upload(p.base, synth.random_bytes(rng, p.size))
    n = 1 << 16
    j = synth.oob_indices(rng, n, p.size // 4, (10 * MiB) // 4, p.size // 4)
    upload(p.base + 4 * MiB, j)
    outs = []
    for mode in ("mask", "modulo"):
        a.gather(p.id, mode, p.base + 6 * MiB, p.base, p.base + 4 * MiB, n)
        outs.append(download(p.base + 6 * MiB, 4 * n))
    assert np.array_equal(outs[0], outs[1])


@pytest.mark.parametrize("mode", ["modulo", "modulo+pa"])
def test_modulo_scatter_near_large_exact_partition(arenas, mode):
    """The scatter-add's near modulo (a table inside a partition of >= 2^33
    bytes: one correction instead of the reciprocal, k_scatter.cu resolve) on
    a non-power-of-two 8 GiB + 14 MiB partition, through the bucketed path,
    with the table 4 GiB into the partition: in-bounds updates, updates past
    the end (offsets in [size + 2 GiB, size + 3 GiB)) and below the base
    (s < 0: the u64 remainder of 2^64 + s, reading A10, which is not the
    Euclidean one for this size).  Every update's word comes from the
    oracle's fence; the partition must equal `before` plus their index_add,
    word for word."""
    import torch
    from paper_2401_09290_b200 import devmem
    GiB = 1 << 30
    size = 8 * GiB + 14 * MiB
    a = arenas(16 * GiB)
    p = a.partition_alloc_exact(size)
    assert p.size == size and not p.pow2
    tab_off, idx_off, src_off = 4 * GiB, GiB, GiB + 8 * MiB

    def addr(j):                                       # table + 4 sext(j), mod 2^64
        return np.uint64(p.base + tab_off) + (4 * np.asarray(j, dtype=np.int64)).astype(np.uint64)

    rng = synth.rng_for(617)
    n = (1 << 20) + 4
    T = 1 << 28                                        # in-bounds words: [4 GiB, 5 GiB)
    j = rng.integers(0, T, n, dtype=np.int64)
    k = synth.planted_count(0.02, n)
    pos = synth.planted_positions(rng, n, k)
    hi, lo = pos[: k // 2], pos[k // 2:]
    j[hi] = (size - 2 * GiB) // 4 + rng.integers(0, GiB // 4, len(hi))        # past the end
    cand = rng.integers(-(1 << 31), -(1 << 30), 8 * len(lo))                    # below the base
    land = oracle.fence_modulo_n(addr(cand), p.base, size, 4) - np.uint64(p.base)
    keep = cand[land >= np.uint64(2 * GiB)]                                      # clear of idx / src
    assert len(keep) >= len(lo)
    j[lo] = keep[: len(lo)]
    off = addr(j) - np.uint64(p.base)
    assert (off[hi] >= np.uint64(size)).all() and (off[lo] > np.uint64(1 << 63)).all()
    jv = j.astype(np.int32)
    src = rng.integers(0, 1 << 32, n, dtype=np.uint64).astype(np.uint32)
    devmem.view(p.base + idx_off, n, torch.int32).copy_(torch.from_numpy(jv))
    devmem.view(p.base + src_off, n, torch.int32).copy_(torch.from_numpy(src.view(np.int32)))
    whole = devmem.view(p.base, size // 4, torch.int32)
    whole[tab_off // 4: tab_off // 4 + T].random_(generator=torch.Generator(device="cuda:0").manual_seed(5))
    before = whole.clone()
    a.stats_reset()
    a.scatter(p.id, mode, p.base + tab_off, p.base + idx_off, p.base + src_off, n)
    assert a.stats(p.id)["violations"] == 0
    words = (oracle.fence_modulo_n(addr(jv), p.base, size, 4) - np.uint64(p.base)) // np.uint64(4)
    w_t = torch.from_numpy(words.astype(np.int64)).cuda()
    s_t = torch.from_numpy(src.astype(np.int64)).cuda()
    u, inv = torch.unique(w_t, return_inverse=True)
    sums = torch.zeros(u.numel(), dtype=torch.int64, device="cuda").index_add_(0, inv, s_t)
    want = (before[u].long() + sums) & 0xFFFFFFFF
    assert torch.equal(whole[u].long() & 0xFFFFFFFF, want)
    after = whole.clone()
    after[u] = before[u]
    assert torch.equal(after, before)
