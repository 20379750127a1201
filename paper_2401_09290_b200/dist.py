"""Multi-GPU plumbing.

Tenants shard naturally: one arena per GPU, a tenant lives on exactly one
GPU, and nothing crosses GPUs on the hot path.  The only collective is the
reduction of the per-GPU statistics (violations / launches / bytes / flops
per tenant and kernel kind) and of the makespan, once per benchmark phase:
``torch.distributed.all_reduce`` over NCCL on GPUs (gloo in the CPU tests).
"""
from __future__ import annotations

import torch
import torch.distributed as dist

FIELDS = ("violations", "launches", "bytes", "flops")


def shard_tenants(n_tenants: int, world: int, rank: int) -> list[int]:
    """Global tenant ids owned by `rank` (round-robin over ranks)."""
    return [t for t in range(n_tenants) if t % world == rank]


def _device():
    if dist.is_initialized() and dist.get_backend() == "nccl":
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device("cpu")


def allreduce_stats(per_tenant: dict[int, dict], makespan_ms: float, n_tenants: int):
    """Sum the per-tenant counters of all ranks and take the max makespan.

    per_tenant: {global tenant id: {"violations": v, "launches": l, "bytes": b, "flops": f}}
    returns ({tenant: {...}}, makespan_ms_max) -- identical on every rank.
    """
    dev = _device()
    vec = torch.zeros(n_tenants * len(FIELDS), dtype=torch.int64, device=dev)
    for t, d in per_tenant.items():
        for k, f in enumerate(FIELDS):
            vec[t * len(FIELDS) + k] = int(d.get(f, 0))
    span = torch.tensor([float(makespan_ms)], dtype=torch.float64, device=dev)
    if dist.is_initialized():
        dist.all_reduce(vec, op=dist.ReduceOp.SUM)
        dist.all_reduce(span, op=dist.ReduceOp.MAX)
    v = vec.cpu().tolist()
    out = {t: {f: v[t * len(FIELDS) + k] for k, f in enumerate(FIELDS)} for t in range(n_tenants)}
    return out, float(span.item())
