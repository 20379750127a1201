"""GPU checks of the C ABI around the kernels: checked host transfers
(§4.2.2), scrubbing on (re)allocation (reading A15), the
trusted counters' placement outside the arena, per-kind stats,
and the partition fill used for the address-revealing pattern."""
import ctypes

import numpy as np
import pytest
import torch

import synth
from paper_2401_09290_b200 import guardian as g
from tests.gpu_util import download, upload

pytestmark = pytest.mark.gpu
MiB = 1 << 20


def test_checked_transfers(arenas):
    a = arenas(4 * MiB)
    p, q = a.partition_alloc(MiB), a.partition_alloc(MiB)
    host = torch.arange(65536, dtype=torch.int32).pin_memory()
    a.memcpy_h2d(p.id, p.base + 4096, host.data_ptr(), 4 * 65536)
    torch.cuda.synchronize()
    assert np.array_equal(download(p.base + 4096, 4 * 65536).view(np.int32), np.arange(65536, dtype=np.int32))
    back = torch.zeros(65536, dtype=torch.int32).pin_memory()
    a.memcpy_d2h(p.id, back.data_ptr(), p.base + 4096, 4 * 65536)
    torch.cuda.synchronize()
    assert torch.equal(back, host)
    qbefore = download(q.base, q.size)
    for dst, n in ((p.end - 8, 16), (q.base, 16), (p.base - 4, 8), (2**64 - 8, 16)):
        with pytest.raises(g.GuardianError) as e:
            a.memcpy_h2d(p.id, dst, host.data_ptr(), n)
        assert e.value.status == g.GD_ERR_OOB_RANGE
    with pytest.raises(g.GuardianError) as e:
        a.memcpy_d2h(p.id, back.data_ptr(), q.base, 64)          # reading the neighbour is refused too
    assert e.value.status == g.GD_ERR_OOB_RANGE
    assert np.array_equal(download(q.base, q.size), qbefore)
    a.memcpy_h2d(p.id, p.end - 16, host.data_ptr(), 16)          # ending exactly at end is fine
    a.memcpy_d2d(p.id, p.base + 8192 * 16, p.base + 4096, 4096)
    torch.cuda.synchronize()
    assert np.array_equal(download(p.base + 8192 * 16, 4096), download(p.base + 4096, 4096))
    for dst, src in ((q.base, p.base), (p.base, q.base), (p.end - 8, p.base)):
        with pytest.raises(g.GuardianError) as e:
            a.memcpy_d2d(p.id, dst, src, 64)
        assert e.value.status == g.GD_ERR_OOB_RANGE


def test_partitions_are_scrubbed_on_reuse(arenas):
    a = arenas(4 * MiB)
    p = a.partition_alloc(MiB)
    upload(p.base, synth.random_bytes(synth.rng_for(1), MiB))
    a.partition_free(p.id)
    q = a.partition_alloc(MiB)
    assert q.base == p.base
    assert not download(q.base, q.size).any()                    # no leak from the previous tenant


def test_stats_live_outside_arena_and_count_per_kind(arenas):
    a = arenas(4 * MiB)
    p = a.partition_alloc(MiB)
    sp = a.stats_device_ptr()
    assert sp + 8 * g.GD_MAX_TENANTS * g.GD_NUM_KINDS <= a.base or sp >= a.base + a.size
    a.stats_reset()
    a.copy(p.id, "check", p.base, p.base + MiB, 64)                # src outside: 4 refused loads
    a.gather(p.id, "check", p.base + 4096, p.base, p.base + 8192, 4)
    st = a.stats(p.id)
    assert st["violations_by_kind"]["copy"] == 4
    assert st["launches_by_kind"]["copy"] == 1 and st["launches_by_kind"]["gather"] == 1
    assert st["bytes"] == 2 * 64 + (4 + 8) * 4
    a.stats_reset(p.id)
    assert a.stats(p.id)["violations"] == 0


def test_partition_fill_pattern(arenas):
    a = arenas(4 * MiB)
    p = a.partition_alloc(MiB)
    a.fill(p.id, 1, 4096, 65536)
    got = download(p.base + 4096, 65536).view(np.uint32)
    np.testing.assert_array_equal(got, synth.pattern_words(np.arange(4096, 4096 + 65536, 4, dtype=np.uint64)))
    with pytest.raises(g.GuardianError) as e:
        a.fill(p.id, 1, MiB - 16, 32)
    assert e.value.status == g.GD_ERR_OOB_RANGE


def test_streams_from_torch_and_async(arenas):
    """Launches are asynchronous on the caller's torch stream."""
    a = arenas(64 * MiB)
    p = a.partition_alloc(32 * MiB)
    s = torch.cuda.Stream()
    upload(p.base, synth.random_bytes(synth.rng_for(2), 8 * MiB))
    torch.cuda.synchronize()
    with torch.cuda.stream(s):
        a.copy(p.id, "mask", p.base + 16 * MiB, p.base, 8 * MiB, stream=s)
    s.synchronize()
    assert np.array_equal(download(p.base + 16 * MiB, 8 * MiB), download(p.base, 8 * MiB))
    assert a.device_flags() == 0


@pytest.mark.parametrize("mode", ["none", "mask", "check", "modulo", "maskcount", "clamp"])
def test_degenerate_launches_do_nothing(arenas, mode):
    """Empty and degenerate shapes (n = 0 is GD_OK and does
    nothing): no byte of the arena changes and nothing is counted, in every
    mode -- including pointers far outside the partition, which an empty
    launch must not even fence."""
    a = arenas(2 * 16 * MiB)
    parts = [a.partition_alloc(16 * MiB) for _ in range(2)]
    for p in parts:
        upload(p.base, np.full(p.size, 0xA5, np.uint8))
    before = download(a.base, a.size)
    p, far = parts[1], 1 << 46
    a.stats_reset()
    a.copy(p.id, mode, far, far, 0)
    a.saxpy(p.id, mode, 2.0, far, far, 0)
    a.gather(p.id, mode, far, far, far, 0)
    a.gather(p.id, mode, far, far, far, 0, 32)
    a.scatter(p.id, mode, far, far, far, 0)
    a.stencil(p.id, mode, far, far, 2, 100, 100, 0.5, 0.125)       # H < 3: no interior point
    a.stencil(p.id, mode, far, far, 100, 2, 100, 0.5, 0.125)       # W < 3
    a.gemm(p.id, mode, far, far, far, 0, 256, 64, 64, 64, 256)       # M = 0
    a.gemm(p.id, mode, far, far, far, 128, 0, 64, 64, 64, 64)        # N = 0
    torch.cuda.synchronize()
    assert np.array_equal(download(a.base, a.size), before)
    assert a.stats(p.id)["violations"] == 0


def test_wrap_caller_owned_torch_memory():
    """gd_arena_wrap over a torch allocation (the caller
    keeps the tensor alive, the library never frees it): partitions carve the
    borrowed range, are scrubbed, and fence like VMM partitions (mask copy
    crossing the end wraps to the partition start, bit-exact vs the oracle)."""
    import oracle
    S = 16 * MiB
    buf = torch.empty(2 * S, dtype=torch.uint8, device="cuda")
    base = (buf.data_ptr() + S - 1) & ~(S - 1)
    with g.Arena.wrap(0, base, S) as a:
        parts = [a.partition_alloc(S // 4) for _ in range(4)]
        assert [p.base for p in parts] == [base + t * (S // 4) for t in range(4)]
        assert (download(base, S) == 0).all()                      # scrubbed (reading A15)
        rng = synth.rng_for(77)
        p = parts[2]
        data = synth.random_bytes(rng, 1 * MiB)
        src = p.base + MiB                          # away from [base, base + over), where the tail wraps
        upload(src, data)
        before = download(base, S)
        n, over = 512 * 1024 + 48, 4096 + 32
        dst = p.end - (n - over)
        a.copy(p.id, "mask", dst, src, n)
        torch.cuda.synchronize()
        mem = oracle.Mem(p.base, buf=before[p.base - base:p.base - base + p.size].copy())
        oracle.copy(mem, p.base, p.size, "mask", dst, src, n)
        after = download(base, S)
        assert np.array_equal(after[p.base - base:p.base - base + p.size], mem.buf)
        lo, hi = p.base - base, p.base - base + p.size
        assert np.array_equal(after[:lo], before[:lo]) and np.array_equal(after[hi:], before[hi:])
    del buf


def test_native_when_solo():
    """with native-when-solo on, a tenant alone runs the native
    kernel (no fence, nothing counted); a second live partition restores
    fencing.  Run on a wrapped torch buffer so that the unfenced access lands
    in mapped (unallocated) arena memory, never outside the allocation."""
    S = 16 * MiB
    buf = torch.empty(2 * S, dtype=torch.uint8, device="cuda")
    base = (buf.data_ptr() + S - 1) & ~(S - 1)
    with g.Arena.wrap(0, base, S) as a:
        a.set_native_when_solo(True)
        p = a.partition_alloc(S // 4)                                  # [base, base + 4 MiB)
        beyond = S // 2                                               # byte offset in the unallocated half
        upload(base + beyond, np.arange(1024, dtype=np.uint32))
        j = np.array([(beyond // 4) + 7, 3], dtype=np.int32)          # one index past the partition
        upload(p.base + MiB, j)
        a.stats_reset()
        a.gather(p.id, "check", p.base + 2 * MiB, p.base, p.base + MiB, 2)
        out = download(p.base + 2 * MiB, 8).view(np.uint32)
        assert out[0] == 7 and a.stats(p.id)["violations"] == 0     # native: read through, not counted
        q = a.partition_alloc(S // 4)                                  # a second tenant arrives
        a.stats_reset()
        a.gather(p.id, "check", p.base + 2 * MiB, p.base, p.base + MiB, 2)
        out = download(p.base + 2 * MiB, 8).view(np.uint32)
        assert out[0] == 0 and a.stats(p.id)["violations"] == 1     # fenced again: refused, counted
        a.partition_free(q.id)
        a.set_native_when_solo(False)
        a.stats_reset()
        a.gather(p.id, "check", p.base + 2 * MiB, p.base, p.base + MiB, 2)
        assert a.stats(p.id)["violations"] == 1                      # off: fenced even when alone
    del buf


def test_launches_and_partition_changes_from_two_threads(arenas):
    """partition alloc / free never run between a launch's
    bounds snapshot and its enqueue.  One thread issues fenced copies into its
    partition while another allocates and frees a neighbour as fast as it
    can; no launch may fault (a stale base would hit unmapped memory) and the
    copies stay correct."""
    import threading
    a = arenas(64 * MiB)
    p = a.partition_alloc(8 * MiB)
    src = np.arange(MiB // 4, dtype=np.uint32)
    upload(p.base, src)
    s = torch.cuda.Stream()
    stop = threading.Event()
    errors = []

    def churn():
        try:
            while not stop.is_set():
                q = a.partition_alloc(8 * MiB)
                a.partition_free(q.id)
        except Exception as e:          # noqa: BLE001
            errors.append(e)

    t = threading.Thread(target=churn)
    t.start()
    try:
        for k in range(2000):
            a.copy(p.id, "check", p.base + MiB * (1 + k % 6), p.base, MiB, stream=s)
    finally:
        stop.set()
        t.join()
    s.synchronize()
    assert not errors, errors
    assert a.stats(p.id)["violations"] == 0
    for k in range(1, 7):
        assert np.array_equal(download(p.base + k * MiB, MiB).view(np.uint32), src)
