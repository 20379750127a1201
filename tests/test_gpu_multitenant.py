"""Multi-tenant launcher on the GPU (SURVEY.md §8(a) a10, config C5 scaled to
a parity-testable size): 8 tenants share one arena and one context, each on
its own stream, issued round-robin by gd_launcher_run.  Tenants 0-2 copy,
3-5 gather with 1 % planted out-of-partition indices, 6-7 GEMM; R launches
each.  Every partition must equal the oracle's simulation of that tenant run
alone (spatial sharing changes nothing a tenant can observe, PAPER.md:230,
258), and the check-mode violations must equal 3 x planted x R."""
import numpy as np
import pytest
import torch

import oracle
import synth
from paper_2401_09290_b200 import guardian as g
from tests.gpu_util import download, first_diff, upload

pytestmark = pytest.mark.gpu

MiB = 1 << 20
PART = 16 * MiB
R = 3
N_IDX, T_N = 1 << 16, 1 << 20
PAT_LO = 10 * MiB


def _bf16_f32(b):
    return (b.astype(np.uint32) << 16).view(np.float32).astype(np.float64)


@pytest.mark.parametrize("policy", ["round_robin", "no_tensor_random", "memory_lane"])
@pytest.mark.parametrize("mode", ["mask", "check"])
def test_c5_mixed_tenants(arenas, mode, policy):
    a = arenas(8 * PART)
    parts = [a.partition_alloc(PART) for _ in range(8)]
    rng = synth.rng_for(5000)
    items, planted = [], 0
    gemm_shape = (256, 256, 256)
    for t, p in enumerate(parts):
        upload(p.base, synth.random_bytes(rng, PART))
        if t < 3:
            items.append(g.work(p.id, g.GD_KIND_COPY, mode, ptr=(p.base + 8 * MiB, p.base + MiB), u64=(3 * MiB + 7,)))
        elif t < 6:
            j = rng.integers(0, T_N, N_IDX, dtype=np.int64).astype(np.int32)
            k = synth.planted_count(0.01, N_IDX)
            pos = synth.planted_positions(rng, N_IDX, k)
            j[pos] = synth.oob_indices(rng, k, PART // 4, PAT_LO // 4, PART // 4)
            planted += k
            upload(p.base + 4 * MiB, j)
            items.append(g.work(p.id, g.GD_KIND_GATHER, mode, ptr=(p.base + 6 * MiB, p.base, p.base + 4 * MiB),
                                u64=(N_IDX,), u32=(1,)))
        else:
            M, N, K = gemm_shape
            upload(p.base, synth.bf16_bits_uniform(rng, M * K))
            upload(p.base + MiB, synth.bf16_bits_uniform(rng, N * K))
            items.append(g.work(p.id, g.GD_KIND_GEMM, mode, ptr=(p.base + 2 * MiB, p.base, p.base + MiB),
                                u64=(K, K, N), u32=(M, N, K)))
    before = download(a.base, a.size)
    queue = [it for it in items for _ in range(R)]            # R launches per tenant, FIFO per tenant
    streams = [torch.cuda.Stream() for _ in parts]
    a.stats_reset()
    order = a.launcher_run(queue, streams, policy=policy)
    tenants_in_order = [queue[i].tenant for i in order]
    assert tenants_in_order[:8] == list(range(8))               # round robin: one per tenant per round
    torch.cuda.synchronize()
    st = a.stats()
    assert st["launches"] == 8 * R
    assert st["violations"] == (planted * R if mode == "check" else 0), (st, planted)   # planted: 3 tenants
    after = download(a.base, a.size)
    for t, p in enumerate(parts):
        lo = p.base - a.base
        mem = oracle.Mem(p.base, buf=before[lo:lo + PART].copy())
        it = items[t]
        for _ in range(R):
            if t < 3:
                oracle.copy(mem, p.base, PART, mode, it.ptr[0], it.ptr[1], it.u64[0])
            elif t < 6:
                oracle.gather(mem, p.base, PART, mode, it.ptr[0], it.ptr[1], it.ptr[2], it.u64[0], 1)
            else:
                M, N, K = gemm_shape
                oracle.gemm(mem, p.base, PART, mode, it.ptr[0], it.ptr[1], it.ptr[2], M, N, K, K, K, N)
        got = after[lo:lo + PART]
        if t < 6:
            assert np.array_equal(got, mem.buf), f"tenant {t}: {first_diff(got, mem.buf)}"
        else:
            M, N, K = gemm_shape
            c0 = 2 * MiB
            cm = np.zeros(PART, bool)
            cm[c0:c0 + 2 * M * N] = True
            assert np.array_equal(got[~cm], mem.buf[~cm])
            gg, rr = _bf16_f32(got[cm].view(np.uint16)), _bf16_f32(mem.buf[cm].view(np.uint16))
            assert np.linalg.norm(gg - rr) / np.linalg.norm(rr) <= 1e-2


def test_solo_vs_shared_victims_identical(arenas):
    """Fault isolation: an attacker tenant whose gather
    indices all point into its neighbours changes nothing they can observe:
    each victim's partition after the shared run equals its solo run."""
    def run(shared: bool):
        a = arenas(4 * PART)
        parts = [a.partition_alloc(PART) for _ in range(4)]
        rng = synth.rng_for(5100)
        for p in parts:
            upload(p.base, synth.random_bytes(rng, PART))
        victims = [g.work(p.id, g.GD_KIND_COPY, "mask", ptr=(p.base + 8 * MiB, p.base + MiB), u64=(2 * MiB,))
                   for p in parts[1:]]
        atk = parts[0]
        j = (np.arange(N_IDX, dtype=np.int64) % 4096 + (PART // 4) * rng.integers(1, 4, N_IDX)).astype(np.int32)
        upload(atk.base + 4 * MiB, j)                         # every raw address in a victim's partition
        attack = [g.work(atk.id, g.GD_KIND_SCATTER, "mask", ptr=(atk.base, atk.base + 4 * MiB, atk.base + 6 * MiB),
                         u64=(N_IDX,))]
        items = victims + (attack * 4 if shared else [])
        a.launcher_run(items, [torch.cuda.Stream() for _ in range(4)])
        torch.cuda.synchronize()
        return [download(p.base, PART) for p in parts[1:]]
    solo, shared = run(False), run(True)
    for v, (x, y) in enumerate(zip(solo, shared)):
        assert np.array_equal(x, y), f"victim {v + 1} differs: {first_diff(x, y)}"
