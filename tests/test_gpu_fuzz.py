"""Seeded fuzz of every kernel against the oracle (whole partition byte for
byte, victims untouched, counts exact).

* check mode: operands anywhere around the partition -- below the base,
  straddling either edge, inside, past the end -- because refused accesses
  never happen, every such input is race-free;
* every other mode: random in-partition shapes and offsets (the fence is the
  identity there, so the result must equal the unfenced twin's).
Sizes are small and ragged (odd lengths, tails, partial tiles)."""
import numpy as np
import pytest

import oracle
import synth
from tests.gpu_util import upload
from tests.test_gpu_kernels import MiB, PART, _run, _setup

pytestmark = pytest.mark.gpu

MODES = ["none", "mask", "check", "modulo", "maskcount", "clamp"]


def _ptr(rng, p, nbytes, align, anywhere):
    """An operand address: inside the partition, or (anywhere) also below,
    straddling either edge or past the end."""
    if anywhere:
        kind = rng.integers(0, 5)
        if kind == 0:
            a = p.base - int(rng.integers(1, 4 * MiB))
        elif kind == 1:
            a = p.base - int(rng.integers(0, max(1, nbytes)))
        elif kind == 2:
            a = p.end - int(rng.integers(0, max(1, nbytes)))
        elif kind == 3:
            a = p.end + int(rng.integers(0, 4 * MiB))
        else:
            a = p.base + int(rng.integers(0, PART - nbytes))
    else:
        a = p.base + int(rng.integers(0, PART - nbytes))
    return a - a % align


def _regions_disjoint(*spans):
    s = sorted(spans)
    return all(a1 <= b0 for (_, a1), (b0, _) in zip(s, s[1:]))


@pytest.mark.parametrize("seed", range(12))
def test_fuzz_streams(arenas, seed):
    a, parts, rng = _setup(arenas, seed=900 + seed)
    p = parts[1]
    for case in range(6):
        mode = MODES[int(rng.integers(0, len(MODES)))]
        anywhere = mode == "check"
        kind = ["copy", "saxpy"][case % 2]
        if kind == "copy":
            n = int(rng.integers(0, 3 * MiB))
            while True:
                src, dst = _ptr(rng, p, n, 16, anywhere), _ptr(rng, p, n, 16, anywhere)
                if _regions_disjoint((src, src + n), (dst, dst + n)):
                    break
            _run(a, parts, 1, mode, lambda p: a.copy(p.id, mode, dst, src, n),
                 lambda m, p: oracle.copy(m, p.base, p.size, mode, dst, src, n))
        else:
            n = int(rng.integers(1, MiB // 2))
            while True:
                x, y = _ptr(rng, p, 4 * n, 16, anywhere), _ptr(rng, p, 4 * n, 16, anywhere)
                if _regions_disjoint((x, x + 4 * n), (y, y + 4 * n)):
                    break
            for q in (x, y):                               # finite floats wherever they land inside
                lo, hi = max(q, p.base), min(q + 4 * n, p.end)
                if hi > lo:
                    upload(lo, synth.uniform_f32(rng, (hi - lo) // 4))
            _run(a, parts, 1, mode, lambda p: a.saxpy(p.id, mode, 0.75, x, y, n),
                 lambda m, p: oracle.saxpy(m, p.base, p.size, mode, 0.75, x, y, n))


@pytest.mark.parametrize("seed", range(12))
def test_fuzz_index(arenas, seed):
    a, parts, rng = _setup(arenas, seed=950 + seed)
    p = parts[2]
    for case in range(6):
        mode = MODES[int(rng.integers(0, len(MODES)))]
        D = int([1, 1, 2, 4, 8, 12, 32, 64, 128, 3][int(rng.integers(0, 10))])
        n = int(rng.integers(0, 20000 if D < 32 else 2000))
        tab = p.base + 16 * int(rng.integers(0, 1024))
        rows = (2 * MiB) // (4 * D)
        j = rng.integers(0, rows, max(n, 1), dtype=np.int64)[:n]
        if mode == "check" and n:
            # any int32 whose row lies wholly outside the partition (a refused
            # access never happens; one landing inside could race with `out`)
            pos = synth.planted_positions(rng, n, max(1, n // 50))
            cand = rng.integers(-2**31, 2**31 - 1, 8 * len(pos))
            ra = tab + 4 * D * cand
            cand = cand[(ra + 4 * D <= p.base) | (ra >= p.end)]
            j[pos] = cand[:len(pos)]
        idx, out = p.base + 4 * MiB, p.base + 8 * MiB
        upload(idx, j.astype(np.int32))
        if case % 2 == 0:
            _run(a, parts, 2, mode, lambda p: a.gather(p.id, mode, out, tab, idx, n, D),
                 lambda m, p: oracle.gather(m, p.base, p.size, mode, out, tab, idx, n, D))
        else:
            src = p.base + 12 * MiB
            jj = j % (2 * MiB // 4)                                      # scatter: word indices
            if mode == "check" and n:
                cand = rng.integers(-2**31, 2**31 - 1, 8 * len(pos))
                ra = tab + 4 * cand
                cand = cand[(ra + 4 <= p.base) | (ra >= p.end)]
                jj[pos] = cand[:len(pos)]
            upload(idx, jj.astype(np.int32))
            upload(src, rng.integers(0, 2**32, max(n, 1), dtype=np.uint64).astype(np.uint32))
            _run(a, parts, 2, mode, lambda p: a.scatter(p.id, mode, tab, idx, src, n),
                 lambda m, p: oracle.scatter_add(m, p.base, p.size, mode, tab, idx, src, n))


@pytest.mark.parametrize("seed", range(8))
def test_fuzz_stencils(arenas, seed):
    a, parts, rng = _setup(arenas, seed=980 + seed)
    p = parts[1]
    for case in range(4):
        mode = MODES[int(rng.integers(0, len(MODES)))]
        anywhere = mode == "check"
        H = int(rng.integers(1, 300))
        W = int(rng.integers(1, 700))
        pitch = W + (-W) % 4 + 4 * int(rng.integers(0, 3))
        nbytes = 4 * H * pitch
        while True:
            inp, out = _ptr(rng, p, nbytes, 16, anywhere), _ptr(rng, p, nbytes, 16, anywhere)
            if _regions_disjoint((inp, inp + nbytes), (out, out + nbytes)):
                break
        lo, hi = max(inp, p.base), min(inp + nbytes, p.end)
        if hi > lo:
            upload(lo, synth.uniform_f32(rng, (hi - lo) // 4, 0.0, 1.0))
        if case % 2 == 0:
            _run(a, parts, 1, mode, lambda p: a.stencil(p.id, mode, out, inp, H, W, pitch, 0.5, 0.125),
                 lambda m, p: oracle.stencil(m, p.base, p.size, mode, out, inp, H, W, pitch, 0.5, 0.125))
        else:
            _run(a, parts, 1, mode, lambda p: a.stencil_tma(p.id, mode, out, inp, H, W, pitch, 0.5, 0.125),
                 lambda m, p: oracle.stencil_tma(m, p.base, p.size, mode, out, inp, H, W, pitch, 0.5, 0.125))
