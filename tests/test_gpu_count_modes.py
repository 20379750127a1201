"""GPU parity of the two counting variants against the CPU oracle:

* maskcount -- mask fencing plus detection: data equal to
  mask mode's, violations equal to check mode's;
* clamp -- north_star's "compare, clamp and set a violation flag" (A1's
  saturating variant): out-of-partition accesses go to the nearest legal
  address at or below them (the base or the last word), counted.

Every clamped store of a 4-byte element lands on one edge word, so clamp-mode
inputs keep out-of-partition accesses to loads and atomics (deterministic),
plus copies whose colliding edge stores carry identical bytes (reading
R-race).  Whole partitions are compared byte for byte with the oracle, the
victims must be untouched, and violation counts exact (tests/test_gpu_kernels
helpers).
"""
import numpy as np
import pytest

import oracle
import synth
from tests.gpu_util import download, upload
from tests.test_gpu_kernels import IDX_OFF, OUT_OFF, PART, PAT_LO, TAB_N, MiB, _gather_inputs, _run, _setup

pytestmark = pytest.mark.gpu

CMODES = ["maskcount", "clamp"]


@pytest.mark.parametrize("mode", CMODES)
@pytest.mark.parametrize("n", [5, 3 * MiB + 16 * 37 + 11])
def test_copy_in_bounds(arenas, mode, n):
    a, parts, _ = _setup(arenas, seed=61)
    _run(a, parts, 1, mode,
         lambda p: a.copy(p.id, mode, p.base + 8 * MiB, p.base + MiB, n),
         lambda m, p: oracle.copy(m, p.base, p.size, mode, p.base + 8 * MiB, p.base + MiB, n), 0)


@pytest.mark.parametrize("mode", CMODES)
def test_copy_from_victim(arenas, mode):
    """src in the partition below: mask-count reads the own partition at the
    wrapped offset, clamp reads the own first 16 bytes for every unit;
    each unit (and tail byte) counted."""
    a, parts, _ = _setup(arenas, seed=62)
    n = MiB + 48 + 5
    _run(a, parts, 1, mode,
         lambda p: a.copy(p.id, mode, p.base + 8 * MiB, parts[0].base + 2 * MiB, n),
         lambda m, p: oracle.copy(m, p.base, p.size, mode, p.base + 8 * MiB, parts[0].base + 2 * MiB, n),
         (n // 16) + n % 16)


@pytest.mark.parametrize("mode", CMODES)
def test_copy_crossing_end(arenas, mode):
    """dst's last units past end.  mask-count: they wrap to [base, base+over)
    like mask mode; clamp: they all land on the last 16 bytes -- the copied
    bytes are made identical for those units, so the collision is benign."""
    a, parts, rng = _setup(arenas, seed=63)
    p = parts[2]
    n, over = 2 * MiB + 16 * 5, 16 * 40
    src = p.base + 1 * MiB
    data = synth.random_bytes(rng, n)
    if mode == "clamp":
        tail = data[n - over - 16:n - over].copy()       # the last in-partition unit
        data[n - over:] = np.tile(tail, over // 16)
    upload(src, data)
    dst = p.end - (n - over)
    _run(a, parts, 2, mode,
         lambda p: a.copy(p.id, mode, dst, src, n),
         lambda m, p: oracle.copy(m, p.base, p.size, mode, dst, src, n), over // 16)


@pytest.mark.parametrize("mode", CMODES)
def test_saxpy_x_crossing_end(arenas, mode):
    """x's last elements lie past end (loads only): mask-count reads the wrapped
    words at the partition start, clamp reads the last word for each; y stays
    inside.  Counted per element."""
    a, parts, rng = _setup(arenas, seed=64)
    p = parts[3]
    n, over = (1 << 18) + 7, 1000 + 3
    x = p.end - 4 * (n - over)
    y = p.base + 1 * MiB
    upload(x, synth.uniform_f32(rng, n - over))
    upload(p.base, synth.uniform_f32(rng, over + 16))          # finite words where x wraps to
    upload(y, synth.uniform_f32(rng, n))
    _run(a, parts, 3, mode,
         lambda p: a.saxpy(p.id, mode, -0.75, x, y, n),
         lambda m, p: oracle.saxpy(m, p.base, p.size, mode, -0.75, x, y, n), over)


def test_saxpy_y_crossing_end_maskcount(arenas):
    a, parts, rng = _setup(arenas, seed=65)
    n, over = (1 << 19) + 7, (1 << 16) + 3
    x = 1 * MiB
    p = parts[3]
    upload(p.base + x, synth.uniform_f32(rng, n))
    y = p.end - 4 * (n - over)
    upload(y, synth.uniform_f32(rng, n - over))
    upload(p.base, synth.uniform_f32(rng, over))
    _run(a, parts, 3, "maskcount",
         lambda p: a.saxpy(p.id, "maskcount", -0.75, p.base + x, y, n),
         lambda m, p: oracle.saxpy(m, p.base, p.size, "maskcount", -0.75, p.base + x, y, n), 2 * over)


@pytest.mark.parametrize("mode", CMODES)
@pytest.mark.parametrize("frac", [0.01, 0.1])
def test_gather_adversarial(arenas, mode, frac):
    a, parts, rng = _setup(arenas, seed=66)
    n = (1 << 18) + 1
    p = parts[2]
    j, pos = _gather_inputs(rng, n, frac)
    upload(p.base + IDX_OFF, j)
    _run(a, parts, 2, mode,
         lambda p: a.gather(p.id, mode, p.base + OUT_OFF, p.base, p.base + IDX_OFF, n),
         lambda m, p: oracle.gather(m, p.base, p.size, mode, p.base + OUT_OFF, p.base, p.base + IDX_OFF, n),
         len(pos))


@pytest.mark.parametrize("mode", CMODES)
@pytest.mark.parametrize("D", [3, 8, 32, 36, 64, 128, 136])
def test_gather_rows_planted_and_straddling(arenas, mode, D):
    """Rows wholly outside (planted), rows straddling the partition end and
    base: every out-of-partition word counted; clamp reads the edge words."""
    a, parts, rng = _setup(arenas, seed=67)
    n = 3000 + D
    tab_off = 48
    j = rng.integers(0, TAB_N // D - 1, n, dtype=np.int64)
    j_hi = (PART - tab_off) // (4 * D)
    pos = synth.planted_positions(rng, n, 96)
    j[pos[0::3]] = j_hi
    j[pos[1::3]] = -1
    far = pos[2::3]
    if mode == "clamp":
        j[far] = rng.integers(-(2**31) // D, -(PART // (4 * D)) - 2, len(far))        # far below: base word
    else:
        # mask-count wraps far rows: their images stay in [PAT_LO, PART) (race-free)
        j[far] = _gather_inputs(rng, len(far), 1.0, D)[0]
    j = j.astype(np.int32)
    upload(parts[1].base + IDX_OFF, j)
    _run(a, parts, 1, mode,
         lambda p: a.gather(p.id, mode, p.base + OUT_OFF, p.base + tab_off, p.base + IDX_OFF, n, D),
         lambda m, p: oracle.gather(m, p.base, p.size, mode, p.base + OUT_OFF, p.base + tab_off,
                                    p.base + IDX_OFF, n, D))


@pytest.mark.parametrize("mode", CMODES)
def test_scatter_add_adversarial(arenas, mode):
    """RMWs outside: mask-count wraps them (into the pattern region), clamp
    piles them on the first / last word -- atomics, so order-independent."""
    a, parts, rng = _setup(arenas, seed=68)
    n = (1 << 18) + 2
    p = parts[1]
    j = rng.integers(0, 4096, n, dtype=np.int64).astype(np.int32)
    k = synth.planted_count(0.05, n)
    pos = synth.planted_positions(rng, n, k)
    j[pos] = synth.oob_indices(rng, k, PART // 4, PAT_LO // 4, PART // 4)
    upload(p.base + IDX_OFF, j)
    _run(a, parts, 1, mode,
         lambda p: a.scatter(p.id, mode, p.base, p.base + IDX_OFF, p.base + OUT_OFF, n),
         lambda m, p: oracle.scatter_add(m, p.base, p.size, mode, p.base, p.base + IDX_OFF, p.base + OUT_OFF, n),
         k)


@pytest.mark.parametrize("mode", CMODES)
@pytest.mark.parametrize("H,W,pitch", [(67, 203, 208), (130, 4, 4)])
def test_stencil_in_bounds(arenas, mode, H, W, pitch):
    a, parts, rng = _setup(arenas, seed=69)
    p = parts[1]
    upload(p.base + MiB, synth.uniform_f32(rng, H * pitch, 0.0, 1.0))
    _run(a, parts, 1, mode,
         lambda p: a.stencil(p.id, mode, p.base + 8 * MiB, p.base + MiB, H, W, pitch, 0.5, 0.125),
         lambda m, p: oracle.stencil(m, p.base, p.size, mode, p.base + 8 * MiB, p.base + MiB, H, W, pitch,
                                     0.5, 0.125), 0)


@pytest.mark.parametrize("mode", CMODES)
def test_stencil_in_crossing_end(arenas, mode):
    """in's last rows lie past end (loads only): mask-count wraps them to the
    partition start, clamp reads the last word for each; counted per logical
    load (5 per interior point, as the oracle)."""
    a, parts, rng = _setup(arenas, seed=70)
    H, W, pitch = 150, 997, 1000
    p = parts[2]
    inp = p.end - (H - 7) * pitch * 4
    upload(inp, synth.uniform_f32(rng, (H - 7) * pitch, 0.0, 1.0))
    upload(p.base, synth.uniform_f32(rng, 8 * pitch, 0.0, 1.0))      # finite words where rows wrap to
    _run(a, parts, 2, mode,
         lambda p: a.stencil(p.id, mode, p.base + 4 * MiB, inp, H, W, pitch, 0.5, 0.125),
         lambda m, p: oracle.stencil(m, p.base, p.size, mode, p.base + 4 * MiB, inp, H, W, pitch, 0.5, 0.125))


def test_stencil_out_crossing_end_maskcount(arenas):
    a, parts, rng = _setup(arenas, seed=71)
    H, W, pitch = 200, 1000, 1024
    p = parts[2]
    upload(p.base + 4 * MiB, synth.uniform_f32(rng, H * pitch, 0.0, 1.0))
    out = p.end - (H - 9) * pitch * 4
    _run(a, parts, 2, "maskcount",
         lambda p: a.stencil(p.id, "maskcount", out, p.base + 4 * MiB, H, W, pitch, 0.5, 0.125),
         lambda m, p: oracle.stencil(m, p.base, p.size, "maskcount", out, p.base + 4 * MiB, H, W, pitch, 0.5,
                                     0.125), 8 * (W - 2))


@pytest.mark.parametrize("mode", CMODES)
def test_c1_toy_counts_655(arenas, mode):
    """BASELINE configs[0] on the 1 MiB VMM arena: bit-exact whole arena and
    exactly the 655 planted violations in both counting variants.  In clamp
    mode an index above the partition reads its last word, which is the last
    word of `out` and written by the same launch (C1 fills the partition):
    those outputs are race-exposed (reading R-race) and excluded, counted."""
    from tests.test_gpu_kernels import _toy_upload
    a = arenas(synth.C1_ARENA)
    parts = [a.partition_alloc(synth.C1_PART) for _ in range(synth.C1_TENANTS)]
    toy = synth.toy_gather()
    host = _toy_upload(a, parts, toy)
    mem = oracle.Mem(a.base, buf=host.copy())
    a.stats_reset()
    total = 0
    for p in parts:
        a.gather(p.id, mode, p.base + synth.C1_OUT_OFF, p.base + synth.C1_TABLE_OFF, p.base + synth.C1_IDX_OFF,
                 synth.C1_N)
        total += oracle.gather(mem, p.base, p.size, mode, p.base + synth.C1_OUT_OFF, p.base + synth.C1_TABLE_OFF,
                               p.base + synth.C1_IDX_OFF, synth.C1_N).violations
    got = download(a.base, a.size)
    keep = np.ones(a.size, bool)
    exposed = 0
    if mode == "clamp":
        for t, p in enumerate(parts):
            raw = p.base + synth.C1_TABLE_OFF + 4 * toy.idx[t].astype(np.int64)
            hi = np.nonzero(raw > p.end - 4)[0]
            exposed += hi.size
            for i in hi:
                o = p.base - a.base + synth.C1_OUT_OFF + 4 * int(i)
                keep[o:o + 4] = False
        assert 0 < exposed < 655
    assert np.array_equal(got[keep], mem.buf[keep])
    print(f"C1 {mode}: {exposed} race-exposed outputs excluded")
    assert total == 655 and sum(a.stats(p.id)["violations"] for p in parts) == 655
