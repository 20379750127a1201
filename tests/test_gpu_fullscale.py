"""GPU parity at the BASELINE.json sizes, in the launch configuration bench.py
and tools/kernel_bench.py time: 16 GiB partitions, C2 (4 GiB copy, 2^30
saxpy), C3 (2^26 indices into a 2^29-entry table, 1 % OOB), C4 (32768^2
stencil, 8192^3 GEMM).

The oracle cannot simulate 16 GiB partitions whole, so each test checks
(a) the exact check-mode violation count (the generator's planted count),
(b) outputs the oracle computes one by one on sampled positions, and
(c) properties that hold at any size (victims unchanged, in-bounds results
equal a library routine, wrapped reads equal the address-revealing pattern's
closed form).
"""
import numpy as np
import pytest
import torch

import oracle
import synth
from paper_2401_09290_b200 import devmem
from tests.gpu_util import download

pytestmark = pytest.mark.gpu

GiB = 1 << 30
PART = 1 << 34
N_IDX, T_N = 1 << 26, 1 << 29
IDX_OFF, OUT_OFF, PAT_OFF = 2 * GiB, 2 * GiB + GiB // 4, 2 * GiB + GiB // 2


@pytest.fixture
def two_tenants(arenas):
    a = arenas(2 * PART)
    victim = a.partition_alloc(PART)
    p = a.partition_alloc(PART)
    assert p.base == victim.base + PART              # raw j < 0 addresses land in the victim
    return a, victim, p


def _c3_inputs(a, p, seed, frac):
    gen = torch.Generator(device="cuda:0")
    gen.manual_seed(seed)
    devmem.view(p.base, T_N, torch.int32).random_(generator=gen)                 # table
    devmem.view(p.base + OUT_OFF, N_IDX, torch.int32).random_(generator=gen)     # out / src
    a.fill(p.id, 1, PAT_OFF, PART - PAT_OFF)                                     # P(o) pattern
    idx, pos = synth.indices_with_oob(synth.rng_for(seed), N_IDX, T_N, frac)
    devmem.view(p.base + IDX_OFF, N_IDX, torch.int32).copy_(torch.from_numpy(idx))
    torch.cuda.synchronize()
    return idx, pos


@pytest.mark.parametrize("mode", ["mask", "check", "maskcount", "clamp", "modulo",
                                  "check+pa", "maskcount+pa", "clamp+pa", "modulo+pa"])
def test_c3_gather_full(two_tenants, mode):
    a, victim, p = two_tenants
    gen = torch.Generator(device="cuda:0")
    gen.manual_seed(3)
    vview = devmem.view(victim.base, PART // 4, torch.int32)
    vview.random_(generator=gen)
    vcopy = vview.clone()
    idx, pos = _c3_inputs(a, p, 3001, 0.01)
    assert len(pos) == 671089
    a.stats_reset()
    a.gather(p.id, mode, p.base + OUT_OFF, p.base, p.base + IDX_OFF, N_IDX)
    st = a.stats(p.id)
    out = devmem.view(p.base + OUT_OFF, N_IDX, torch.int32)
    table = devmem.view(p.base, T_N, torch.int32)
    idx_t = devmem.view(p.base + IDX_OFF, N_IDX, torch.int32).long()
    inb = torch.ones(N_IDX, dtype=torch.bool, device="cuda")
    pos_t = torch.from_numpy(pos).cuda()
    inb[pos_t] = False
    # (c) in-bounds results equal index_select; victims untouched
    assert torch.equal(out[inb], table[idx_t[inb]])
    assert torch.equal(vview, vcopy)
    # (a) + (c) planted positions (modulo on a pow2 partition wraps like mask)
    base_mode = mode.split("+")[0]
    if base_mode == "check":
        assert st["violations"] == 671089
        assert (out[pos_t] == 0).all()
    elif base_mode == "clamp":                   # every planted j < 0 lands below the base: word 0
        assert st["violations"] == 671089
        assert (out[pos_t] == table[0]).all()
    else:
        assert st["violations"] == (671089 if base_mode == "maskcount" else 0)
        j = idx[pos].astype(np.int64)
        expect = synth.pattern_words(np.mod(PART + 4 * j, PART).astype(np.uint64)).view(np.int32)
        np.testing.assert_array_equal(out[pos_t].cpu().numpy(), expect)
    # (b) oracle, one by one, on sampled positions (planted and in-bounds)
    rng = synth.rng_for(7)
    sample = np.concatenate([rng.choice(pos, 2000, replace=False), rng.integers(0, N_IDX, 2000)])
    outs = out.cpu().numpy()
    for i in sample:
        ai, ok = oracle.resolve(p.base, p.size, base_mode, p.base + IDX_OFF + 4 * int(i), 4)
        assert ok and ai == p.base + IDX_OFF + 4 * int(i)
        r, ok = oracle.resolve(p.base, p.size, base_mode, (p.base + 4 * int(idx[i])) % 2**64, 4)
        want = 0 if not ok else int(download(r, 4).view(np.int32)[0])
        assert outs[i] == want, (i, idx[i], outs[i], want)


ROW_TAB_OFF, ROW_IDX_OFF, ROW_OUT_OFF, ROW_PAT_OFF = 0, 2 * GiB + GiB // 2, 3 * GiB, 4 * GiB


@pytest.mark.parametrize("D", [32, 6])          # k_gatherR (128-bit row slots) / k_gatherE (flat words)
@pytest.mark.parametrize("mode", ["mask", "check", "maskcount", "clamp", "modulo",
                                  "check+pa", "modulo+pa", "clamp+pa"])
def test_row_gather_full(two_tenants, mode, D):
    """The row gathers in tools/kernel_bench.py's and bench.py's configuration:
    a 2^29-word table viewed as rows of D words, 1 GiB of gathered rows,
    1 % planted rows at j in [-2^20, 0) (below the base; mask / modulo wrap
    them into the top 128 MiB of the partition, which holds the pattern)."""
    a, victim, p = two_tenants
    rows, n = T_N // D, GiB // (4 * D)
    gen = torch.Generator(device="cuda:0")
    gen.manual_seed(40 + D)
    devmem.view(p.base + ROW_TAB_OFF, T_N, torch.int32).random_(generator=gen)
    devmem.view(p.base + ROW_OUT_OFF, n * D, torch.int32).random_(generator=gen)
    a.fill(p.id, 1, ROW_PAT_OFF, PART - ROW_PAT_OFF)
    rng = synth.rng_for(4000 + D)
    j = rng.integers(0, rows, n, dtype=np.int64)
    pos = synth.planted_positions(rng, n, synth.planted_count(0.01, n))
    j[pos] = rng.integers(-(1 << 20), 0, len(pos), dtype=np.int64)
    j = j.astype(np.int32)
    devmem.view(p.base + ROW_IDX_OFF, n, torch.int32).copy_(torch.from_numpy(j))
    vview = devmem.view(victim.base, GiB // 4, torch.int32)
    vcopy = vview.clone()
    torch.cuda.synchronize()
    a.stats_reset()
    a.gather(p.id, mode, p.base + ROW_OUT_OFF, p.base + ROW_TAB_OFF, p.base + ROW_IDX_OFF, n, D)
    st = a.stats(p.id)
    out = devmem.view(p.base + ROW_OUT_OFF, n * D, torch.int32).view(n, D)
    table = devmem.view(p.base + ROW_TAB_OFF, T_N, torch.int32)[: rows * D].view(rows, D)
    j_t = torch.from_numpy(j.astype(np.int64)).cuda()
    inb = torch.ones(n, dtype=torch.bool, device="cuda")
    pos_t = torch.from_numpy(pos).cuda()
    inb[pos_t] = False
    # (c) in-bounds rows equal index_select; the victim below is untouched
    assert torch.equal(out[inb], table[j_t[inb]])
    assert torch.equal(vview, vcopy)
    # (a) + (c) planted rows
    base_mode = mode.split("+")[0]
    if base_mode == "check":
        assert st["violations"] == len(pos) * D
        assert (out[pos_t] == 0).all()
    elif base_mode == "clamp":                   # every word of a planted row lies below the base: word 0
        assert st["violations"] == len(pos) * D
        assert (out[pos_t] == table[0, 0]).all()
    else:
        assert st["violations"] == (len(pos) * D if base_mode == "maskcount" else 0)
        o = np.mod(PART + 4 * (j[pos].astype(np.int64)[:, None] * D + np.arange(D)[None, :]), PART)
        assert (o >= ROW_PAT_OFF).all()
        np.testing.assert_array_equal(out[pos_t].cpu().numpy(), synth.pattern_words(o.astype(np.uint64)).view(np.int32))
    # (b) oracle, one access at a time, on sampled words (planted and in-bounds rows)
    srng = synth.rng_for(8 + D)
    rows_s = np.concatenate([srng.choice(pos, 300, replace=False), srng.integers(0, n, 300)])
    cols_s = srng.integers(0, D, len(rows_s))
    outs = out.cpu().numpy()
    for i, d in zip(rows_s, cols_s):
        a_t = (p.base + ROW_TAB_OFF + 4 * (int(j[i]) * D + int(d))) % 2**64
        r, ok = oracle.resolve(p.base, p.size, base_mode, a_t, 4)
        want = 0 if not ok else int(download(r, 4).view(np.int32)[0])
        assert outs[i, d] == want, (i, d, j[i], outs[i, d], want)


@pytest.mark.parametrize("mode", ["mask", "check", "maskcount", "clamp", "modulo",
                                  "check+pa", "maskcount+pa", "clamp+pa", "modulo+pa"])
def test_c3_scatter_full(two_tenants, mode):
    a, victim, p = two_tenants
    idx, pos = _c3_inputs(a, p, 3002, 0.01)
    before = devmem.view(p.base, PART // 4, torch.int32).clone()
    a.stats_reset()
    a.scatter(p.id, mode, p.base, p.base + IDX_OFF, p.base + OUT_OFF, N_IDX)
    st = a.stats(p.id)
    mode = mode.split("+")[0]                     # per access: the same results and counts
    assert st["violations"] == (0 if mode in ("mask", "modulo") else 671089)
    after = devmem.view(p.base, PART // 4, torch.int32)
    src = devmem.view(p.base + OUT_OFF, N_IDX, torch.int32).long() & 0xFFFFFFFF
    idx_t = torch.from_numpy(idx.astype(np.int64)).cuda()
    inb = torch.ones(N_IDX, dtype=torch.bool, device="cuda")
    pos_t = torch.from_numpy(pos).cuda()
    inb[pos_t] = False
    # table region: index_add_ reference (int64, reduced mod 2^32)
    ref = before[:T_N].long() & 0xFFFFFFFF
    ref.index_add_(0, idx_t[inb], src[inb])
    if mode == "clamp":                          # every planted j < 0 clamps to word 0 (sums per CTA, exact)
        ref[0] += src[pos_t].sum()
    assert torch.equal(after[:T_N].long() & 0xFFFFFFFF, ref & 0xFFFFFFFF)
    del ref
    if mode in ("mask", "maskcount", "modulo"):
        # planted indices: the oracle fences each raw address; the adds land there
        # (modulo on a pow2 partition wraps like mask)
        raw = (p.base + 4 * idx[pos].astype(np.int64)).astype(np.uint64)
        f = oracle.fence_mask_n(raw, p.base, p.size, 4)
        words = torch.from_numpy(((f - np.uint64(p.base)) // np.uint64(4)).astype(np.int64)).cuda()
        assert (words >= T_N).all()
        u, inv = torch.unique(words, return_inverse=True)
        sums = torch.zeros(u.numel(), dtype=torch.int64, device="cuda").index_add_(0, inv, src[pos_t])
        want = (before[u].long() + sums) & 0xFFFFFFFF
        assert torch.equal(after[u].long() & 0xFFFFFFFF, want)
        after[u] = before[u]                         # then nothing else may differ
    assert torch.equal(after[T_N:], before[T_N:])


@pytest.mark.parametrize("mode", ["mask", "none", "check", "modulo", "maskcount", "clamp",
                                  "check+pa", "modulo+pa", "maskcount+pa", "clamp+pa"])
def test_c2_copy_saxpy_full(arenas, mode):
    """C2 at the bench's size and launch configuration (one 16 GiB partition,
    4 GiB copy, 2^30-element saxpy: k_copy / k_saxpy with 262,144 CTAs), in
    every mode, hoisted and per access (+pa): the copy equals its source
    byte for byte, and 2^20 seeded saxpy elements equal the oracle's, bit
    for bit; nothing is counted (every access is inside)."""
    a = arenas(PART)
    p = a.partition_alloc(PART)
    gen = torch.Generator(device="cuda:0")
    gen.manual_seed(2000)
    src = devmem.view(p.base, GiB, torch.int32)
    src.random_(generator=gen)
    x = devmem.view(p.base + 8 * GiB, 1 << 30, torch.float32)
    y = devmem.view(p.base + 12 * GiB, 1 << 30, torch.float32)
    x.uniform_(-1, 1, generator=gen)
    y.uniform_(-1, 1, generator=gen)
    rng = synth.rng_for(8)
    s = torch.from_numpy(rng.integers(0, 1 << 30, 1 << 20)).cuda()
    xs, ys = x[s].cpu().numpy(), y[s].cpu().numpy()
    a.stats_reset()
    a.copy(p.id, mode, p.base + 4 * GiB, p.base, 4 * GiB)
    a.saxpy(p.id, mode, 1.5, p.base + 8 * GiB, p.base + 12 * GiB, 1 << 30)
    assert a.stats(p.id)["violations"] == 0
    assert torch.equal(devmem.view(p.base + 4 * GiB, GiB, torch.int32), src)
    got = y[s].cpu().numpy()
    m = oracle.Mem(0x10000000, 8 << 20)
    m.write(0x10000000, xs)
    m.write(0x10000000 + (4 << 20), ys)
    oracle.saxpy(m, 0x10000000, 8 << 20, mode.split("+")[0], 1.5, 0x10000000, 0x10000000 + (4 << 20), 1 << 20)
    np.testing.assert_array_equal(got.view(np.uint32), m.view(0x10000000 + (4 << 20), np.uint32, 1 << 20))


@pytest.mark.parametrize("mode", ["mask", "check", "modulo", "maskcount", "clamp"])
def test_c2_full_crossing_end(arenas, mode):
    """SURVEY.md §8(d) C2 parity variant at the bench size: src / x at 4 GiB,
    dst / y at 12 GiB + 1 MiB, so the last 1 MiB of dst / y crosses the end of
    the 16 GiB partition (the >= 4 GiB mask path, kMaskBig, walks into it).
    Mask / modulo / mask-count wrap it into offsets [0, 1 MiB), which nothing
    else touches (race-free); check refuses and counts it (65,536 16-byte
    stores; 2 x 262,144 y accesses); clamp counts like check.  Checked: the
    whole wrapped MiB and the last inside MiB of the copy, the counts, and
    2^20 sampled saxpy elements plus every wrapped one against the oracle."""
    a = arenas(PART)
    p = a.partition_alloc(PART)
    MiB = 1 << 20
    src = x = p.base + 4 * GiB
    dst = y = p.base + 12 * GiB + MiB
    n = 1 << 30
    gen = torch.Generator(device="cuda:0")
    gen.manual_seed(2003)
    devmem.view(src, GiB, torch.int32).random_(generator=gen)
    devmem.view(p.base, MiB // 4, torch.float32).uniform_(-1, 1, generator=gen)       # the wrap target
    wrap0 = download(p.base, MiB)
    counting = mode in ("check", "maskcount", "clamp")
    # copy
    a.stats_reset()
    a.copy(p.id, mode, dst, src, 4 * GiB)
    assert a.stats(p.id)["violations"] == (MiB // 16 if counting else 0)
    tail_in = download(src + 4 * GiB - 2 * MiB, 2 * MiB)          # the source of the last inside / outside MiB
    last_in = download(p.end - MiB, MiB)
    if mode == "clamp":       # the last 16-byte unit: the copy's clamped unit stores collide there (R-race)
        np.testing.assert_array_equal(last_in[:-16], tail_in[:MiB - 16])
    else:
        np.testing.assert_array_equal(last_in, tail_in[:MiB])
    wrapped = download(p.base, MiB)
    if mode in ("mask", "modulo", "maskcount"):
        np.testing.assert_array_equal(wrapped, tail_in[MiB:])
    elif mode == "check":
        np.testing.assert_array_equal(wrapped, wrap0)             # nothing landed
    # saxpy (x = the copy's source as floats: finite values are all that matters;
    # y starts as what the copy wrote inside and as wrap0 wrapped)
    devmem.view(x, n, torch.float32).uniform_(-1, 1, generator=gen)
    devmem.view(y, n - MiB // 4, torch.float32).uniform_(-1, 1, generator=gen)
    devmem.view(p.base, MiB // 4, torch.float32).uniform_(-1, 1, generator=gen)
    xv = devmem.view(x, n, torch.float32)
    yv_in = devmem.view(y, n - MiB // 4, torch.float32)
    rng = synth.rng_for(11)
    s_in = torch.from_numpy(np.unique(np.concatenate([rng.integers(0, n - MiB // 4, 1 << 20),
                                                      np.arange(n - MiB // 4 - 4096, n - MiB // 4)]))).cuda()
    if mode == "clamp":
        s_in = s_in[s_in != n - MiB // 4 - 1]                      # the edge word: clamped stores collide (R-race)
    xs, ys = xv[s_in].cpu().numpy(), yv_in[s_in].cpu().numpy()
    x_tail = xv[n - MiB // 4:].cpu().numpy()
    y_wrap0 = download(p.base, MiB).view(np.float32).copy()
    a.stats_reset()
    a.saxpy(p.id, mode, 1.5, x, y, n)
    assert a.stats(p.id)["violations"] == (2 * (MiB // 4) if counting else 0)

    def oracle_saxpy(xa, ya):
        k = xa.size
        m = oracle.Mem(0x10000000, 8 * k + 64)
        m.write(0x10000000, xa)
        m.write(0x10000000 + 4 * k, ya)
        oracle.saxpy(m, 0x10000000, 8 * k + 64, "none", 1.5, 0x10000000, 0x10000000 + 4 * k, k)
        return m.view(0x10000000 + 4 * k, np.uint32, k)

    np.testing.assert_array_equal(yv_in[s_in].cpu().numpy().view(np.uint32), oracle_saxpy(xs, ys))
    got_wrap = download(p.base, MiB).view(np.uint32)
    if mode in ("mask", "modulo", "maskcount"):
        np.testing.assert_array_equal(got_wrap, oracle_saxpy(x_tail, y_wrap0))
    elif mode == "check":
        np.testing.assert_array_equal(got_wrap, y_wrap0.view(np.uint32))


def test_c4_stencil_full_sampled_rows(arenas):
    a = arenas(PART)
    p = a.partition_alloc(PART)
    H = W = 32768
    inp, out = p.base + 4 * GiB, p.base + 8 * GiB
    gen = torch.Generator(device="cuda:0")
    gen.manual_seed(4000)
    devmem.view(inp, H * W, torch.float32).uniform_(0, 1, generator=gen)
    a.stencil(p.id, "mask", out, inp, H, W, W, 0.5, 0.125)
    rng = synth.rng_for(9)
    rows = np.concatenate([[1, 2, 63, 64, 65, H - 2], rng.integers(1, H - 1, 20)])
    for r in rows:
        band = download(inp + 4 * (int(r) - 1) * W, 3 * 4 * W)
        m = oracle.Mem(0x20000000, 4 << 20)
        m.buf[:band.size] = band
        oracle.stencil(m, 0x20000000, 4 << 20, "none", 0x20000000 + (2 << 20), 0x20000000, 3, W, W, 0.5, 0.125)
        want = m.view(0x20000000 + (2 << 20) + 4 * W, np.uint32, W)[1:W - 1]
        got = download(out + 4 * int(r) * W, 4 * W).view(np.uint32)[1:W - 1]
        np.testing.assert_array_equal(got, want, err_msg=f"row {r}")


@pytest.mark.parametrize("mode", ["mask", "check", "modulo", "maskcount"])
def test_c4_stencil_full_out_crossing_end(arenas, mode):
    """SURVEY.md §8(d) C4 adversarial layout at the bench size: `out` at
    end - (H-64)·pitch·4, so its last 64 rows lie past the end.  Mask /
    modulo wrap them into offsets [0, 64·pitch·4) (untouched otherwise, so
    the run is race-free); check refuses and counts their 63·(W-2) interior
    stores; mask-count stores like mask and counts like check.  Sampled rows
    (inside, the first crossing row, the last) against the oracle's 3-row
    band.  Run hoisted here and per access (k_stencil_pa, the modulo walk)
    by test_gpu_peraccess.py."""
    a = arenas(PART)
    p = a.partition_alloc(PART)
    H = W = 32768
    inp, out = p.base + 4 * GiB, p.end - (H - 64) * W * 4
    gen = torch.Generator(device="cuda:0")
    gen.manual_seed(4001)
    devmem.view(inp, H * W, torch.float32).uniform_(0, 1, generator=gen)
    a.stats_reset()
    a.stencil(p.id, mode, out, inp, H, W, W, 0.5, 0.125)
    v = a.stats(p.id)["violations"]
    assert v == (63 * (W - 2) if mode in ("check", "maskcount") else 0)
    rows = [1, 2, 1000, H - 66, H - 65, H - 64, H - 63, H - 3, H - 2]
    for r in rows:
        band = download(inp + 4 * (r - 1) * W, 3 * 4 * W)
        m = oracle.Mem(0x20000000, 4 << 20)
        m.buf[:band.size] = band
        oracle.stencil(m, 0x20000000, 4 << 20, "none", 0x20000000 + (2 << 20), 0x20000000, 3, W, W, 0.5, 0.125)
        want = m.view(0x20000000 + (2 << 20) + 4 * W, np.uint32, W)[1:W - 1]
        dst = out + 4 * r * W
        inside = dst + 4 * W <= p.end
        if not inside:
            dst = p.base + (dst - p.base) % p.size          # mask = modulo on a pow2 partition
        got = download(dst, 4 * W).view(np.uint32)[1:W - 1]
        if inside or mode in ("mask", "modulo", "maskcount"):
            np.testing.assert_array_equal(got, want, err_msg=f"row {r}")
        else:
            assert not got.any(), f"row {r}: a refused store landed"     # scrubbed, never written


@pytest.mark.parametrize("mode", ["mask", "check", "modulo", "maskcount", "clamp"])
def test_c4_stencil_full_in_crossing_end(arenas, mode):
    """The input side of the C4 layout at the bench size: `in` at
    end - (H-64)·pitch·4, so its rows H-64 .. H-1 lie wholly past the end
    (16 GiB partition: the >= 4 GiB path of the stencil, incl. check mode's
    masked loads with their zero fix-up when run per access by
    test_gpu_peraccess.py).  Each point's five loads resolve per the mode:
    mask / modulo / mask-count read the row wrapped to offset
    (4·x·W + in - base) mod size (filled with random floats), check reads 0,
    clamp reads the partition's last word (fence.cuh edge4); the counting
    modes count (W-2)·(64 + 3·63 + 62) refused loads (N of rows >= H-63, C/W/E
    of rows >= H-64, S of rows >= H-65).  Sampled rows against the oracle's
    stencil over the 3-row band built that way."""
    a = arenas(PART)
    p = a.partition_alloc(PART)
    H = W = 32768
    inp, out = p.end - (H - 64) * W * 4, p.base + 4 * GiB
    gen = torch.Generator(device="cuda:0")
    gen.manual_seed(4002)
    devmem.view(inp, (H - 64) * W, torch.float32).uniform_(0, 1, generator=gen)
    devmem.view(p.base, 64 * W, torch.float32).uniform_(0, 1, generator=gen)     # the wrap target
    torch.cuda.synchronize()
    a.stats_reset()
    a.stencil(p.id, mode, out, inp, H, W, W, 0.5, 0.125)
    v = a.stats(p.id)["violations"]
    assert v == ((W - 2) * (64 + 3 * 63 + 62) if mode in ("check", "maskcount", "clamp") else 0)
    last = download(p.end - 4, 4)                                                # clamp's edge word

    def in_row(x):
        addr = inp + 4 * x * W
        if addr + 4 * W <= p.end:
            return download(addr, 4 * W)
        if mode == "check":
            return np.zeros(4 * W, np.uint8)
        if mode == "clamp":
            return np.tile(last, W)
        return download(p.base + (addr - p.base) % p.size, 4 * W)               # mask = modulo (pow2)

    for r in [1, 1000, H - 67, H - 66, H - 65, H - 64, H - 63, H - 3, H - 2]:
        band = np.concatenate([in_row(x) for x in (r - 1, r, r + 1)])
        m = oracle.Mem(0x20000000, 4 << 20)
        m.buf[:band.size] = band
        oracle.stencil(m, 0x20000000, 4 << 20, "none", 0x20000000 + (2 << 20), 0x20000000, 3, W, W, 0.5, 0.125)
        want = m.view(0x20000000 + (2 << 20) + 4 * W, np.uint32, W)[1:W - 1]
        got = download(out + 4 * r * W, 4 * W).view(np.uint32)[1:W - 1]
        np.testing.assert_array_equal(got, want, err_msg=f"row {r}")


@pytest.mark.parametrize("side", ["in", "out"])
@pytest.mark.parametrize("mode", ["mask", "check", "modulo", "maskcount", "clamp"])
def test_stencil_small_grid_big_partition_crossing(arenas, side, mode):
    """The L2-resident size (2048^2: 8-row strips) in a 16 GiB partition, so
    the >= 4 GiB code paths of the small-grid kernels run (one-LOP3 partition
    test, mask fence on the high word walking fenced pointers, mask-count's
    BIG variant), with `in` or `out` crossing the partition end by 64 rows:
    EVERY row against the oracle's stencil over its 3-row band (resolved per
    mode as in test_c4_stencil_full_in_crossing_end; a refused or wrapped
    output row as in test_c4_stencil_full_out_crossing_end), and the exact
    count.  Hoisted here, per access via test_gpu_peraccess.py."""
    a = arenas(PART)
    p = a.partition_alloc(PART)
    H = W = 2048
    rb = 4 * W
    if side == "in":
        inp, out = p.end - (H - 64) * rb, p.base + 4 * GiB
    else:
        inp, out = p.base + 4 * GiB, p.end - (H - 64) * rb
    gen = torch.Generator(device="cuda:0")
    gen.manual_seed(4003)
    n_in = (H - 64) * W if side == "in" else H * W
    devmem.view(inp, n_in, torch.float32).uniform_(0, 1, generator=gen)
    devmem.view(p.base, 64 * W, torch.float32).uniform_(0, 1, generator=gen)       # wrap target of `in`
    torch.cuda.synchronize()
    a.stats_reset()
    a.stencil(p.id, mode, out, inp, H, W, W, 0.5, 0.125)
    v = a.stats(p.id)["violations"]
    counting = mode in ("check", "maskcount", "clamp")
    if side == "in":
        assert v == ((W - 2) * (64 + 3 * 63 + 62) if counting else 0)
    else:
        assert v == (63 * (W - 2) if counting else 0)
    inside_in = download(inp, n_in * 4)                                          # the rows inside
    wrap = download(p.base, 64 * rb)
    last = download(p.end - 4, 4)

    def in_row(x):
        if inp + (x + 1) * rb <= p.end:
            return inside_in[x * rb:(x + 1) * rb]
        if mode == "check":
            return np.zeros(rb, np.uint8)
        if mode == "clamp":
            return np.tile(last, W)
        o = (inp + x * rb - p.base) % p.size                                     # mask = modulo (pow2)
        return wrap[o:o + rb]

    for r in range(1, H - 1):
        band = np.concatenate([in_row(x) for x in (r - 1, r, r + 1)])
        m = oracle.Mem(0x20000000, 1 << 16)
        m.buf[:band.size] = band
        oracle.stencil(m, 0x20000000, 1 << 16, "none", 0x20000000 + (1 << 15), 0x20000000, 3, W, W, 0.5, 0.125)
        want = m.view(0x20000000 + (1 << 15) + rb, np.uint32, W)[1:W - 1]
        dst = out + r * rb
        if dst + rb <= p.end:
            got = download(dst, rb).view(np.uint32)[1:W - 1]
            np.testing.assert_array_equal(got, want, err_msg=f"row {r}")
        elif mode in ("mask", "modulo", "maskcount"):
            got = download(p.base + (dst - p.base) % p.size, rb).view(np.uint32)[1:W - 1]
            np.testing.assert_array_equal(got, want, err_msg=f"row {r} (wrapped)")


def test_c4_stencil_v2_full_sampled_rows(arenas):
    """K5 v2 at the BASELINE size in the bench's launch configuration: sampled
    rows (incl. tile edges at 16-row and 248-column boundaries) against the
    oracle's or_stencil_tma on the 3-row band, and the boundary columns kept."""
    a = arenas(PART)
    p = a.partition_alloc(PART)
    H = W = 32768
    inp, out = p.base + 4 * GiB, p.base + 8 * GiB
    gen = torch.Generator(device="cuda:0")
    gen.manual_seed(4001)
    devmem.view(inp, H * W, torch.float32).uniform_(0, 1, generator=gen)
    devmem.view(out, H * W, torch.float32).fill_(-3.0)
    a.stencil_tma(p.id, "mask", out, inp, H, W, W, 0.5, 0.125)
    assert a.device_flags() == 0                                       # no TMA wait expired
    rng = synth.rng_for(10)
    rows = np.concatenate([[1, 2, 16, 17, 18, H - 2], rng.integers(1, H - 1, 20)])
    for r in rows:
        band = download(inp + 4 * (int(r) - 1) * W, 3 * 4 * W)
        m = oracle.Mem(0x20000000, 4 << 20)
        m.buf[:band.size] = band
        oracle.stencil_tma(m, 0x20000000, 4 << 20, "none", 0x20000000 + (2 << 20), 0x20000000, 3, W, W, 0.5, 0.125)
        want = m.view(0x20000000 + (2 << 20) + 4 * W, np.uint32, W)[1:W - 1]
        row = download(out + 4 * int(r) * W, 4 * W).view(np.float32)
        np.testing.assert_array_equal(row.view(np.uint32)[1:W - 1], want, err_msg=f"row {r}")
        assert row[0] == -3.0 and row[W - 1] == -3.0                   # boundary columns untouched
    for r in (0, H - 1):
        assert (download(out + 4 * r * W, 4 * W).view(np.float32) == -3.0).all()


@pytest.mark.parametrize("mode,clamp", [("mask", False), ("check", False), ("check", True), ("mask", True),
                                        ("clamp", True)])
def test_c4_gemm_8192_sampled_rows(arenas, mode, clamp):
    """C4 GEMM at 8192^3 in the bench's launch configuration (2-SM tcgen05,
    persistent), 256 seeded rows of C (incl. the 128-row tile edges, the
    first / last rows and, with `clamp`, the rows around A's end) against the
    oracle's fp64 -> fp32 -> bf16 rows: relative Frobenius <= 1e-2
    (north_star) and element-wise |g - r| <= 2 ulp_bf16(r) + 2^-16 S,
    S = sum_k |a_ik b_jk| (DESIGN.md R-GEMM), so one wrong tile or a dropped
    K slice fails.  clamp: A's last 64 rows lie past the partition end
    (SURVEY §8(d) C4); they read as zero, so those C rows are exactly 0, and
    check / clamp count them (64)."""
    a = arenas(PART)
    p = a.partition_alloc(PART)
    n, MiB = 8192, 1 << 20
    if clamp:                                   # A's last 64 rows lie past end
        A = p.end - (n - 64) * n * 2
        B, C = A - 160 * MiB, A - 320 * MiB
    else:
        A, B, C = p.base, p.base + 160 * MiB, p.base + 320 * MiB
    gen = torch.Generator(device="cuda:0")
    gen.manual_seed(4001)
    devmem.view(A, (n - 64) * n if clamp else n * n, torch.bfloat16).uniform_(-1, 1, generator=gen)
    devmem.view(B, n * n, torch.bfloat16).uniform_(-1, 1, generator=gen)
    a.stats_reset()
    a.gemm(p.id, mode, C, A, B, n, n, n, n, n, n)
    assert a.device_flags() == 0
    assert a.stats(p.id)["violations"] == (64 if clamp and mode in ("check", "clamp") else 0)
    rng = synth.rng_for(10)
    edges = [0, 127, 128, 255, 256, 4095, 4096, n - 129, n - 128, n - 65, n - 64, n - 63, n - 1]
    rows = np.unique(np.concatenate([edges, rng.choice(n, 256 - len(edges), replace=False)]))[:256]
    rows = rows.astype(np.uint32)
    lo = min(A, B, C)
    hi = p.end if clamp else max(A, B, C) + 2 * n * n
    mem = oracle.Mem(lo, buf=download(lo, hi - lo))
    gpu_c = download(C, 2 * n * n).view(np.uint16).reshape(n, n)
    c = oracle.gemm(mem, p.base, p.size, mode, C, A, B, n, n, n, n, n, n, rows=rows)
    assert c.faults == 0
    ref_c = mem.view(C, np.uint16, n * n).reshape(n, n)
    g = (gpu_c[rows].astype(np.uint32) << 16).view(np.float32).astype(np.float64)
    r = (ref_c[rows].astype(np.uint32) << 16).view(np.float32).astype(np.float64)
    rel = np.linalg.norm(g - r) / max(np.linalg.norm(r), 1e-30)
    assert rel <= 1e-2, rel
    # S = |A_rows| |B|^T (rows of A past the end read as zero in every mode here)
    valid = (n - 64) if clamp else n
    a_rows = np.zeros((len(rows), n), np.float32)
    ok = rows < valid
    a_bits = mem.view(A, np.uint16, valid * n).reshape(valid, n)
    a_rows[ok] = np.abs((a_bits[rows[ok]].astype(np.uint32) << 16).view(np.float32))
    b_abs = np.abs((mem.view(B, np.uint16, n * n).astype(np.uint32) << 16).view(np.float32)).reshape(n, n)
    S = (a_rows @ b_abs.T).astype(np.float64)
    from tests.test_gpu_gemm import bf16_ulp
    err = np.abs(g - r)
    bad = err > 2 * bf16_ulp(r) + 2.0 ** -16 * S
    assert not bad.any(), (int(bad.sum()), float(err.max()), [(int(rows[i // n]), i % n) for i in
                                                             np.flatnonzero(bad)[:5]])
    if clamp:
        assert (gpu_c[n - 64:] == 0).all()
