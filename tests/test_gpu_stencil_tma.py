"""GPU parity of K5 v2, the TMA-staged stencil (both operands fenced in their
tensor maps), against the oracle's or_stencil_tma: whole partition byte for
byte, victims untouched, counts exact (tests/test_gpu_kernels helpers)."""
import numpy as np
import pytest

import oracle
import synth
from tests.gpu_util import upload
from tests.test_gpu_kernels import MiB, _run, _setup

pytestmark = pytest.mark.gpu

ALL = ["none", "mask", "check", "modulo", "maskcount", "clamp"]
FENCED = ALL[1:]


@pytest.fixture(autouse=True)
def no_tma_wait_timed_out():
    """k_stencil_tma bounds its mbarrier waits (~2 s, then
    it raises device flag bit 1 and stores nothing); after every K5 v2 test
    the flags must be clear (no wait ever expired)."""
    yield
    from paper_2401_09290_b200 import guardian as g
    with g.Arena(0, 1 << 20) as a:
        assert a.device_flags() == 0


@pytest.mark.parametrize("mode", ALL)
@pytest.mark.parametrize("H,W,pitch", [(3, 3, 4), (67, 203, 208), (300, 1100, 1104), (130, 4, 4), (1030, 509, 512)])
def test_stencil_tma_in_bounds(arenas, mode, H, W, pitch):
    a, parts, rng = _setup(arenas, seed=81)
    p = parts[1]
    upload(p.base + MiB, synth.uniform_f32(rng, H * pitch, 0.0, 1.0))
    _run(a, parts, 1, mode,
         lambda p: a.stencil_tma(p.id, mode, p.base + 8 * MiB, p.base + MiB, H, W, pitch, 0.5, 0.125),
         lambda m, p: oracle.stencil_tma(m, p.base, p.size, mode, p.base + 8 * MiB, p.base + MiB, H, W, pitch,
                                         0.5, 0.125), 0)


@pytest.mark.parametrize("mode", FENCED)
def test_stencil_tma_in_crossing_end(arenas, mode):
    """in's last rows lie past end: TMA reads them as zeros (no wrap in any
    mode); the counting modes count those rows."""
    a, parts, rng = _setup(arenas, seed=82)
    H, W, pitch = 300, 777, 780
    p = parts[2]
    keep = 211
    inp = p.end - keep * pitch * 4
    upload(inp, synth.uniform_f32(rng, keep * pitch, 0.0, 1.0))
    _run(a, parts, 2, mode,
         lambda p: a.stencil_tma(p.id, mode, p.base + 4 * MiB, inp, H, W, pitch, 0.5, 0.125),
         lambda m, p: oracle.stencil_tma(m, p.base, p.size, mode, p.base + 4 * MiB, inp, H, W, pitch, 0.5, 0.125),
         (H - keep) if mode in ("check", "maskcount", "clamp") else 0)


@pytest.mark.parametrize("mode", FENCED)
def test_stencil_tma_out_crossing_end(arenas, mode):
    """out's last rows lie past end (in v2 the TMA clamp
    skips them): those interior points are not stored, nothing wraps."""
    a, parts, rng = _setup(arenas, seed=83)
    H, W, pitch = 200, 1001, 1004                    # 4 (W - 1) = 4000: 16-byte multiple
    p = parts[2]
    upload(p.base + 4 * MiB, synth.uniform_f32(rng, H * pitch, 0.0, 1.0))
    room = 137                                       # rows of out (W - 1 floats) inside
    out = p.end - (room - 1) * 4 * pitch - 4 * (W - 1)
    assert out % 16 == 0
    _run(a, parts, 2, mode,
         lambda p: a.stencil_tma(p.id, mode, out, p.base + 4 * MiB, H, W, pitch, 0.5, 0.125),
         lambda m, p: oracle.stencil_tma(m, p.base, p.size, mode, out, p.base + 4 * MiB, H, W, pitch, 0.5, 0.125),
         (H - 1 - room) if mode in ("check", "maskcount", "clamp") else None)


@pytest.mark.parametrize("mode", ["mask", "check", "clamp", "modulo"])
def test_stencil_tma_in_from_victim(arenas, mode):
    """in points into another tenant: check reads no row (zeros), mask /
    modulo fence the base into the own partition, clamp moves it to the own
    base (the victim lies below)."""
    a, parts, rng = _setup(arenas, seed=84)
    H, W, pitch = 100, 777, 780
    p = parts[1]
    inp = parts[0].base + 2 * MiB
    upload(inp, synth.uniform_f32(rng, H * pitch))
    upload(p.base, synth.uniform_f32(rng, H * pitch))                 # where clamp lands
    upload(p.base + 2 * MiB, synth.uniform_f32(rng, H * pitch))       # where mask / modulo land
    _run(a, parts, 1, mode,
         lambda p: a.stencil_tma(p.id, mode, p.base + 8 * MiB, inp, H, W, pitch, 0.5, 0.125),
         lambda m, p: oracle.stencil_tma(m, p.base, p.size, mode, p.base + 8 * MiB, inp, H, W, pitch, 0.5, 0.125),
         None if mode in ("mask", "modulo") else H)


def test_stencil_tma_equals_v1_inside(arenas):
    """Inside the partition the two variants compute the same bits."""
    a, parts, rng = _setup(arenas, seed=85)
    H, W, pitch = 513, 1300, 1304
    p = parts[1]
    upload(p.base + MiB, synth.uniform_f32(rng, H * pitch, 0.0, 1.0))
    from tests.gpu_util import download
    a.stencil(p.id, "mask", p.base + 8 * MiB, p.base + MiB, H, W, pitch, 0.5, 0.125)
    v1 = download(p.base + 8 * MiB, 4 * H * pitch).copy()
    upload(p.base + 8 * MiB, np.zeros(4 * H * pitch, np.uint8))
    a.stencil_tma(p.id, "mask", p.base + 8 * MiB, p.base + MiB, H, W, pitch, 0.5, 0.125)
    v2 = download(p.base + 8 * MiB, 4 * H * pitch)
    f1 = v1.view(np.float32).reshape(H, pitch)
    f2 = v2.view(np.float32).reshape(H, pitch)
    np.testing.assert_array_equal(f1[1:H - 1, 1:W - 1].view(np.uint32), f2[1:H - 1, 1:W - 1].view(np.uint32))
