"""Captured multi-tenant steps (gd_graph_*): a replay computes exactly what
the launcher computes (bit-exact against the oracle for the C1 toy, in mask
and check mode, violations included), accounting counts every replay, a
graph refuses to replay after any partition it fences was re-allocated, and
for launch-bound steps the replay is cheaper than issuing kernel by kernel."""
import time

import numpy as np
import pytest
import torch

import oracle
import synth
from paper_2401_09290_b200 import guardian as g
from tests.gpu_util import download, first_diff, upload

pytestmark = pytest.mark.gpu


def _toy(arenas):
    a = arenas(synth.C1_ARENA)
    parts = [a.partition_alloc(synth.C1_PART) for _ in range(synth.C1_TENANTS)]
    toy = synth.toy_gather()
    host = np.zeros(a.size, np.uint8)
    for t, p in enumerate(parts):
        o = p.base - a.base
        host[o:o + 4 * synth.C1_TABLE_N] = toy.tables[t].view(np.uint8)
        host[o + synth.C1_IDX_OFF:o + synth.C1_IDX_OFF + 4 * synth.C1_N] = toy.idx[t].view(np.uint8)
    upload(a.base, host)
    return a, parts, toy, host


@pytest.mark.parametrize("mode", ["mask", "check", "maskcount", "modulo"])
def test_graph_replay_matches_oracle(arenas, mode):
    a, parts, toy, host = _toy(arenas)
    items = [g.work(p.id, g.GD_KIND_GATHER, mode, ptr=(p.base + synth.C1_OUT_OFF, p.base, p.base + synth.C1_IDX_OFF),
                    u64=(synth.C1_N,), u32=(1,)) for p in parts]
    graph = a.graph(items, n_streams=4)
    a.stats_reset()
    for _ in range(3):
        graph.launch()
    torch.cuda.synchronize()
    mem = oracle.Mem(a.base, buf=host.copy())
    for p in parts:
        oracle.gather(mem, p.base, p.size, mode, p.base + synth.C1_OUT_OFF, p.base, p.base + synth.C1_IDX_OFF,
                      synth.C1_N)
    got = download(a.base, a.size)
    assert np.array_equal(got, mem.buf), first_diff(got, mem.buf)
    st = a.stats()
    assert st["launches"] == 3 * len(items)
    assert st["violations"] == (3 * toy.n_planted if mode in ("check", "maskcount") else 0)
    graph.close()


def test_graph_refuses_stale_partitions(arenas):
    a, parts, _, _ = _toy(arenas)
    items = [g.work(parts[1].id, g.GD_KIND_COPY, "mask", ptr=(parts[1].base + 4096, parts[1].base), u64=(4096,))]
    graph = a.graph(items, n_streams=1)
    graph.launch()
    a.partition_free(parts[1].id)
    with pytest.raises(g.GuardianError) as e:
        graph.launch()
    assert e.value.status == g.GD_ERR_UNKNOWN_PARTITION
    q = a.partition_alloc(synth.C1_PART)             # same id and base, new generation
    assert q.id == parts[1].id and q.base == parts[1].base
    with pytest.raises(g.GuardianError):
        graph.launch()
    graph.close()


def test_graph_is_cheaper_for_small_steps(arenas):
    """64 tiny fenced kernels across 8 tenants: one graph replay vs 64 calls."""
    a = arenas(8 << 20)
    parts = [a.partition_alloc(1 << 20) for _ in range(8)]
    items = [g.work(p.id, g.GD_KIND_COPY, "mask", ptr=(p.base + 4096 * (k + 1), p.base), u64=(4096,))
             for k in range(8) for p in parts]
    streams = [torch.cuda.Stream() for _ in parts]
    graph = a.graph(items, n_streams=8)
    for _ in range(5):
        a.launcher_run(items, streams)
        graph.launch()
    torch.cuda.synchronize()
    reps = 50
    t0 = time.perf_counter()
    for _ in range(reps):
        a.launcher_run(items, streams)
    torch.cuda.synchronize()
    t_launcher = (time.perf_counter() - t0) / reps
    t0 = time.perf_counter()
    for _ in range(reps):
        graph.launch()
    torch.cuda.synchronize()
    t_graph = (time.perf_counter() - t0) / reps
    print(f"64-kernel step: launcher {t_launcher * 1e6:.1f} us, graph {t_graph * 1e6:.1f} us")
    assert t_graph < t_launcher
    graph.close()


def test_graph_captured_solo_goes_stale():
    """a graph captured while a tenant ran alone with
    native-when-solo holds unfenced kernels, so it may replay only while the
    arena's partition set and the switch are unchanged; a graph of fenced
    kernels keeps replaying while its own partitions stand."""
    MiB = 1 << 20
    S = 16 * MiB
    buf = torch.empty(2 * S, dtype=torch.uint8, device="cuda")
    base = (buf.data_ptr() + S - 1) & ~(S - 1)
    with g.Arena.wrap(0, base, S) as a:
        a.set_native_when_solo(True)
        p = a.partition_alloc(S // 4)
        beyond = S // 2
        upload(base + beyond, np.arange(1024, dtype=np.uint32))
        upload(p.base + MiB, np.array([(beyond // 4) + 7, 3], dtype=np.int32))
        item = g.work(p.id, g.GD_KIND_GATHER, "check", ptr=(p.base + 2 * MiB, p.base, p.base + MiB), u64=(2,),
                      u32=(1,))
        solo = a.graph([item], n_streams=1)
        solo.launch()
        assert download(p.base + 2 * MiB, 8).view(np.uint32)[0] == 7      # native: read through
        q = a.partition_alloc(S // 4)                                      # a second tenant arrives
        with pytest.raises(g.GuardianError) as e:
            solo.launch()
        assert e.value.status == g.GD_ERR_UNKNOWN_PARTITION
        fenced = a.graph([item], n_streams=1)                              # captured fenced (two live)
        a.partition_free(q.id)
        with pytest.raises(g.GuardianError):                               # alone again: still stale
            solo.launch()
        upload(p.base + 2 * MiB, np.zeros(2, np.uint32))
        fenced.launch()                                                    # fenced graph: still valid
        assert download(p.base + 2 * MiB, 8).view(np.uint32)[0] == 0
        solo2 = a.graph([item], n_streams=1)
        a.set_native_when_solo(False)                                      # the switch changes: stale
        with pytest.raises(g.GuardianError):
            solo2.launch()
        for gr in (solo, fenced, solo2):
            gr.close()
    del buf


def test_zero_row_growth_keeps_captured_graphs_valid(arenas):
    """a GEMM whose A has no legal row reads a trusted zero
    row; a later launch that needs a longer row grows it without freeing the
    old one, so a graph captured earlier still reads zeros."""
    a = arenas(64 << 20)
    p = a.partition_alloc(64 << 20)
    M = N = 128
    C, B = p.base, p.base + (1 << 20)
    upload(B, (np.ones((N, 256), np.float32).view(np.uint32) >> 16).astype(np.uint16))
    bad_A = p.base - (4 << 20)                                             # below the base: no legal row
    small = g.work(p.id, g.GD_KIND_GEMM, "check", ptr=(C, bad_A, B), u64=(64, 256, N), u32=(M, N, 64))
    gr = a.graph([small], n_streams=1)
    a.gemm(p.id, "check", C + (8 << 20), bad_A, B, M, N, 256, 256, 256, N)   # K = 256: the zero row grows
    upload(C, np.full(M * N, 0x3F80, np.uint16))                          # C = 1.0 before the replay
    gr.launch()
    torch.cuda.synchronize()
    assert not download(C, 2 * M * N).any()                                # zeros from the old zero row
    assert a.device_flags() == 0
    gr.close()
