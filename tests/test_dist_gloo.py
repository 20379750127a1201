"""The N > 1 path on CPU: world_size 2 over gloo.  Each rank owns a shard of
the C1 tenants, simulates its tenants' check-mode gathers with the oracle, and
the per-tenant statistics are reduced with the same all_reduce the GPUs use
over NCCL.  The reduced violations must equal the planted count (655) and
every tenant must be counted exactly once."""
import os
import socket

import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    import torch.distributed as dist

    import oracle
    import synth
    from paper_2401_09290_b200 import dist as gdist

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    toy = synth.toy_gather()
    arena = 0x7FA2C0000000
    mem = oracle.Mem(arena, synth.C1_ARENA)
    for t in range(synth.C1_TENANTS):
        b = arena + t * synth.C1_PART
        mem.write(b + synth.C1_TABLE_OFF, toy.tables[t])
        mem.write(b + synth.C1_IDX_OFF, toy.idx[t])
    mine = gdist.shard_tenants(synth.C1_TENANTS, world, rank)
    per = {}
    for t in mine:
        b = arena + t * synth.C1_PART
        c = oracle.gather(mem, b, synth.C1_PART, "check", b + synth.C1_OUT_OFF, b + synth.C1_TABLE_OFF,
                          b + synth.C1_IDX_OFF, synth.C1_N, 1)
        per[t] = {"violations": c.violations, "launches": 1, "bytes": 12 * synth.C1_N, "flops": 0}
    red, span = gdist.allreduce_stats(per, makespan_ms=10.0 + rank, n_tenants=synth.C1_TENANTS)
    q.put((rank, mine, red, span))
    dist.destroy_process_group()


def test_gloo_world2_stats_reduce():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    owned = sorted(t for _, mine, _, _ in res for t in mine)
    assert owned == [0, 1, 2, 3]                               # every tenant on exactly one rank
    for _, _, red, span in res:
        assert sum(d["violations"] for d in red.values()) == 655
        assert all(d["launches"] == 1 for d in red.values())
        assert span == 11.0                                    # max over ranks
    assert res[0][2] == res[1][2]
