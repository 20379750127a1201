"""Pins of the oracle's K5 v2 (TMA-staged stencil, both operands
descriptor-fenced: SURVEY.md §2.7 K5, §8(a) a9, §8(c) O2).

* inside the partition: the NumPy slice expression with one exact fused
  rounding (tests/exact.py), independent of the oracle;
* `in` crossing the end: the same expression with the rows past the
  descriptor's row count replaced by zeros (TMA OOB fill), the row count
  found by enumerating rows whose bytes all lie in the partition;
* `out` crossing the end: rows past its row count keep their old bytes;
  row 0, row H-1, column 0 and column W-1 are never written;
* counts: the rows check would refuse, by the same enumeration.
"""
import numpy as np
import pytest

import oracle
import synth
from tests.exact import exact_fma_f32

PBASE, PSIZE = 1 << 30, 1 << 20
C0, C1 = np.float32(0.5), np.float32(0.125)


def _ref(f, H, W):
    """Interior points of the Jacobi sweep over field f (H x >= W), exact fma."""
    s = (f[0:H - 2, 1:W - 1] + f[2:H, 1:W - 1]) + (f[1:H - 1, 0:W - 2] + f[1:H - 1, 2:W])
    t = C0 * f[1:H - 1, 1:W - 1]
    return np.vectorize(lambda si, ti: exact_fma_f32(C1, si, ti), otypes=[np.float32])(s, t)


def _rows_inside(p, rows, rowbytes, stride):
    """Longest prefix of rows whose bytes all lie in [PBASE, PBASE + PSIZE)."""
    if not (PBASE <= p and p + rowbytes <= PBASE + PSIZE):
        return 0
    k = 0
    while k < rows and p + k * stride + rowbytes <= PBASE + PSIZE:
        k += 1
    return k


@pytest.mark.parametrize("mode", ["none", "mask", "check", "modulo", "maskcount", "clamp"])
def test_inside_partition_matches_slices(mode):
    rng = synth.rng_for(71)
    H, W, pitch = 22, 29, 32
    f = synth.uniform_f32(rng, H * pitch, 0.0, 1.0).reshape(H, pitch)
    m = oracle.Mem(PBASE, PSIZE)
    inp, out = PBASE + 4096, PBASE + 65536
    m.write(inp, f.reshape(-1))
    old = synth.random_bytes(rng, 4 * H * pitch)
    m.write(out, old)
    c = oracle.stencil_tma(m, PBASE, PSIZE, mode, out, inp, H, W, pitch, float(C0), float(C1))
    o = m.view(out, np.float32, H * pitch).reshape(H, pitch)
    np.testing.assert_array_equal(o[1:H - 1, 1:W - 1].view(np.uint32), _ref(f, H, W).view(np.uint32))
    ob = old.view(np.float32).reshape(H, pitch)
    for sl in (np.s_[0, :], np.s_[H - 1, :], np.s_[:, 0], np.s_[:, W - 1:]):
        np.testing.assert_array_equal(o[sl].view(np.uint32), ob[sl].view(np.uint32))     # never written
    assert c.violations == 0 and c.faults == 0


@pytest.mark.parametrize("mode", ["mask", "check", "maskcount", "clamp", "modulo"])
def test_in_crossing_end_reads_zero_rows(mode):
    rng = synth.rng_for(72)
    H, W, pitch = 40, 61, 64
    keep = 31                                        # rows of `in` inside the partition
    inp = PBASE + PSIZE - keep * 4 * pitch
    f = synth.uniform_f32(rng, keep * pitch, 0.0, 1.0).reshape(keep, pitch)
    m = oracle.Mem(PBASE, PSIZE)
    m.write(inp, f.reshape(-1))
    out = PBASE + 8192
    c = oracle.stencil_tma(m, PBASE, PSIZE, mode, out, inp, H, W, pitch, float(C0), float(C1))
    rin = _rows_inside(inp, H, 4 * W, 4 * pitch)
    assert rin == keep
    full = np.zeros((H, pitch), np.float32)
    full[:rin] = f[:rin]
    o = m.view(out, np.float32, H * pitch).reshape(H, pitch)
    np.testing.assert_array_equal(o[1:H - 1, 1:W - 1].view(np.uint32), _ref(full, H, W).view(np.uint32))
    counted = mode in ("check", "maskcount", "clamp")
    assert c.violations == (H - rin if counted else 0)


@pytest.mark.parametrize("mode", ["mask", "check", "clamp"])
def test_out_crossing_end_rows_not_stored(mode):
    rng = synth.rng_for(73)
    H, W, pitch = 30, 41, 44                          # 4 (W-1) = 160: `out` stays 16-byte aligned
    f = synth.uniform_f32(rng, H * pitch, 0.0, 1.0).reshape(H, pitch)
    m = oracle.Mem(PBASE, PSIZE)
    inp = PBASE
    m.write(inp, f.reshape(-1))
    room = 17                                        # rows of `out` (W-1 floats each) inside the partition
    out = PBASE + PSIZE - (room - 1) * 4 * pitch - 4 * (W - 1)
    assert out % 16 == 0
    before = m.buf.copy()
    c = oracle.stencil_tma(m, PBASE, PSIZE, mode, out, inp, H, W, pitch, float(C0), float(C1))
    rout = _rows_inside(out, H - 1, 4 * (W - 1), 4 * pitch)
    assert rout == room
    ref = _ref(f, H, W)
    for r in range(1, H - 1):
        a = out + 4 * r * pitch
        for col in (1, W // 2, W - 2):
            x = a + 4 * col
            if r < rout:
                got = m.view(x, np.float32, 1)[0]
                assert got.view(np.uint32) == ref[r - 1, col - 1].view(np.uint32)
            elif x + 4 <= PBASE + PSIZE:
                assert m.view(x, np.uint8, 4).tobytes() == before[x - PBASE:x - PBASE + 4].tobytes()
    assert c.faults == 0
    assert c.violations == ((H - 1) - rout if mode in ("check", "clamp") else 0)


def test_check_in_outside_reads_all_zero():
    """check mode, `in` in another partition: no row may be read; every
    interior output is fmaf(c1, 0, c0 * 0) = +0; all H rows counted."""
    H, W, pitch = 12, 20, 20
    m = oracle.Mem(PBASE, PSIZE)
    out = PBASE + 4096
    m.write(out, np.full(H * pitch, 7.0, np.float32))
    c = oracle.stencil_tma(m, PBASE, PSIZE, "check", out, PBASE - (1 << 20), H, W, pitch, float(C0), float(C1))
    o = m.view(out, np.float32, H * pitch).reshape(H, pitch)
    assert (o[1:H - 1, 1:W - 1] == 0).all() and (o[0] == 7).all() and (o[:, W - 1] == 7).all()
    assert c.violations == H


@pytest.mark.parametrize("mode", ["mask", "check", "clamp", "modulo", "maskcount"])
@pytest.mark.parametrize("shift", [0, 4, 16, 60, 100, 4 * 39, 4 * 41])
def test_out_rows_stored_iff_every_interior_point_inside(mode, shift):
    """Reading R-TMA-out, pinned without the extent formula:
    K5 v2 stores whole rows.  With `out` crossing the partition end, row r's
    interior points are stored iff EVERY interior point of row r lies in the
    partition (byte membership of each 4-byte point, enumerated here), and a
    row that is only partly inside keeps all its old bytes -- unlike v1's
    per-access fence, which stores (mask: wraps) each point on its own.  The
    sweep of `shift` moves the end across every column position of a row."""
    rng = synth.rng_for(74)
    H, W, pitch = 14, 41, 44
    f = synth.uniform_f32(rng, H * pitch, 0.0, 1.0).reshape(H, pitch)
    m = oracle.Mem(PBASE, PSIZE)
    m.write(PBASE, f.reshape(-1))
    out = PBASE + PSIZE - 6 * 4 * pitch - shift            # rows 6.. cross or pass the end
    out -= out % 16
    sentinel = np.full(((PBASE + PSIZE) - out) // 4, 0x7F7F7F7F, np.uint32)
    m.write(out, sentinel)
    oracle.stencil_tma(m, PBASE, PSIZE, mode, out, PBASE, H, W, pitch, float(C0), float(C1))
    ref = _ref(f, H, W)
    end = PBASE + PSIZE
    for r in range(1, H - 1):
        pts = [out + 4 * (r * pitch + col) for col in range(1, W - 1)]
        inside = [all(PBASE <= b < end for b in range(x, x + 4)) for x in pts]
        whole = all(inside)
        for col, x, ins in zip(range(1, W - 1), pts, inside):
            if not ins:
                continue                                   # not in this partition's memory
            got = m.view(x, np.uint32, 1)[0]
            if whole:
                assert got == ref[r - 1, col - 1].view(np.uint32), (r, col)
            else:
                assert got == 0x7F7F7F7F, (r, col)          # partly inside: the row is not stored
