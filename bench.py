#!/usr/bin/env python
"""Benchmark: fenced-kernel HBM GB/s (% of peak) and overhead vs the unfenced twin.

Workload (BASELINE.json configs[1], "C2"): per GPU one 2^37-byte arena with
8 tenants x 16 GiB partitions; every step, the multi-tenant launcher issues,
round-robin over the tenants onto one stream per tenant, each tenant's fenced
streaming copy of 4 GiB and fenced fp32 SAXPY over 2^30 elements (4 GiB
tensors).  value = algorithmic bytes of all tenants on all GPUs / step time.

  python bench.py [--gpus N --steps K --warmup W --mode mask|check|none]
  python bench.py --impl reference      # the CPU oracle on the host cores
  python bench.py --gpus 2 --dry-run    # the rank plumbing on CPU (gloo, virtual arenas)

With --gpus N > 1 and no WORLD_SIZE in the environment, bench.py launches
itself under torch.distributed.run with N ranks; under torchrun WORLD_SIZE
must equal --gpus.  Every rank runs its own arena (tenants shard across
GPUs, no data-path collective); the step time is the max over ranks and the
per-GPU statistics are summed with one NCCL all_reduce.
Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

GiB = 1 << 30
MiB = 1 << 20
# fence modes in gd_mode order; the unfenced twin first (overheads are against it)
ALL_MODES = ("none", "mask", "check", "modulo", "maskcount", "clamp")


def gpu_config(mode, world):
    """The bench line's config (both arms)."""
    return {"workload": WORKLOAD, "mode": mode, "tenants_per_gpu": TENANTS,
            "partition_bytes": PART, "copy_bytes": COPY_BYTES, "saxpy_n": SAXPY_N,
            "l2": "inputs larger than L2 (4 GiB per tensor vs 126 MB L2), no flush",
            "parallelism": f"{world} GPU(s), one arena per GPU, tenants sharded, no data-path collective"}


def paper_mean(xs):
    """The paper's statistic: the mean without the minimum and
    the maximum (of its 10 runs; here of the table's repetitions)."""
    xs = sorted(xs)
    core = xs[1:-1] if len(xs) > 2 else xs
    return sum(core) / len(core)


def rotated(modes, r):
    """The mode order of repetition r: rotated by r, so that over len(modes)
    repetitions every mode runs once in every position of the sequence (a
    kernel's clock under the power cap depends on what ran just before it;
    a fixed order biased the later modes of the 0.5 ms GEMM by up to 5 %)."""
    k = r % len(modes)
    return list(modes[k:]) + list(modes[:k])
TENANTS = 8
PART = 1 << 34                    # 16 GiB
ARENA = TENANTS * PART            # 2^37
COPY_BYTES = 1 << 32              # 4 GiB
SAXPY_N = 1 << 30                 # 2^30 fp32 = 4 GiB per tensor
OFF_SRC, OFF_DST, OFF_X, OFF_Y = 0, 4 * GiB, 8 * GiB, 12 * GiB
ALPHA = 1.5
BYTES_COPY = 2 * COPY_BYTES       # algorithmic bytes per launch
BYTES_SAXPY = 12 * SAXPY_N
STEP_BYTES_PER_GPU = TENANTS * (BYTES_COPY + BYTES_SAXPY)
METRIC = "fenced-kernel HBM GB/s (% of peak) and overhead % vs unfenced, 1/2/4/8 B200"
WORKLOAD = ("C2: 8 tenants x 16 GiB pow2 partitions per GPU; per tenant fenced copy of 4 GiB + fenced fp32 "
            "SAXPY over 2^30 elements, issued round-robin on 8 streams by the native launcher")


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d.get("hbm_gbs", 6650.0)), float(d.get("bf16_tflops", 1590.0)), \
            float(d.get("bf16_tflops_sustained", 1400.0)), "measured"
    return 6650.0, 1590.0, 1400.0, "fallback"


# ---------------------------------------------------------------------------
# clocks sampler (nvidia-smi during the timed region)
# ---------------------------------------------------------------------------

class Clocks:
    FIELDS = ["clocks.sm", "clocks.max.sm", "clocks_event_reasons.hw_slowdown",
              "clocks_event_reasons.hw_thermal_slowdown", "clocks_event_reasons.sw_thermal_slowdown",
              "clocks_event_reasons.sw_power_cap"]

    def __init__(self, device: int):
        self.device, self.rows, self.proc = device, [], None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), "--query-gpu=" + ",".join(self.FIELDS),
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except (OSError, FileNotFoundError):
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) == len(self.FIELDS):
                self.rows.append(parts)

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[2 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "sm_min_mhz": min(sm) if sm else None, "reasons": reasons, "samples": len(self.rows)}


# ---------------------------------------------------------------------------
# distributed plumbing
# ---------------------------------------------------------------------------

_JSON_FD = None


def quiet_stdout():
    """Route everything written to fd 1 (NCCL prints "NCCL version ..." to
    stdout at communicator setup) to stderr; emit() writes the one JSON line
    to the original stdout."""
    global _JSON_FD
    if _JSON_FD is None:
        sys.stdout.flush()
        _JSON_FD = os.dup(1)
        os.dup2(2, 1)


def emit(line):
    data = (json.dumps(line) + "\n").encode()
    if _JSON_FD is None:
        sys.stdout.write(data.decode())
        sys.stdout.flush()
    else:
        sys.stdout.flush()
        os.write(_JSON_FD, data)


def dist_init(backend="nccl"):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # GD_FORCE_DIST=1 brings NCCL up at world size 1 too, so a one-GPU box
    # exercises the collective path (stats all_reduce, max-over-ranks timing)
    if world > 1 or os.environ.get("GD_FORCE_DIST") == "1":
        import torch.distributed as dist
        import torch
        if backend == "nccl":
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
        else:
            dist.init_process_group(backend)
    return world, rank, local


def allreduce(vals, op="max"):
    import torch
    import torch.distributed as dist
    from paper_2401_09290_b200 import dist as gdist
    dev = gdist._device() if dist.is_available() and dist.is_initialized() else \
        torch.device("cuda" if torch.cuda.is_available() else "cpu")
    t = torch.tensor(vals, dtype=torch.float64, device=dev)
    if dist.is_available() and dist.is_initialized():
        dist.all_reduce(t, op=dist.ReduceOp.MAX if op == "max" else dist.ReduceOp.SUM)
    return t.tolist()


def spawn_ranks(args):
    """--gpus N > 1 without WORLD_SIZE: run this script under
    torch.distributed.run with N ranks (one per GPU, 127.0.0.1 rendezvous)
    and pass its exit code and its one JSON line through."""
    import socket
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    r = subprocess.run(cmd, stdout=subprocess.PIPE, text=True)
    sys.stdout.write(r.stdout)
    sys.stdout.flush()
    return r.returncode


def barrier():
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized():
        dist.barrier()


# ---------------------------------------------------------------------------
# the work items (shared by the GPU arm and the dry run)
# ---------------------------------------------------------------------------

C5_N_IDX, C5_TABLE_N, C5_GEMM_N = 1 << 26, 1 << 29, 8192
C5_IDX_OFF, C5_OUT_OFF = 2 * GiB, 2 * GiB + GiB // 4


def c2_items(g, parts, mode):
    """BASELINE configs[1] (C2) step of one GPU: per tenant a fenced copy of
    4 GiB and a fenced SAXPY over 2^30 elements."""
    its = []
    for p in parts:
        its.append(g.work(p.id, g.GD_KIND_COPY, mode, ptr=(p.base + OFF_DST, p.base + OFF_SRC), u64=(COPY_BYTES,)))
        its.append(g.work(p.id, g.GD_KIND_SAXPY, mode, ptr=(p.base + OFF_X, p.base + OFF_Y), u64=(SAXPY_N,),
                          f32=(ALPHA,)))
    return its


def c5_items(g, parts, mode):
    """BASELINE configs[4] (C5) of one GPU: t0-t2 fenced copy (4 GiB), t3-t5
    fenced gather (C3: 2^26 indices into a 2^29-word table), t6-t7 fenced
    GEMM 8192^3.  Returns (items, algorithmic bytes, flops) of one round."""
    n = C5_GEMM_N
    items, nbytes, flops = [], 0, 0
    for t, p in enumerate(parts):
        b = p.base
        if t < 3:
            items.append(g.work(p.id, g.GD_KIND_COPY, mode, ptr=(b + OFF_DST, b + OFF_SRC), u64=(COPY_BYTES,)))
            nbytes += BYTES_COPY
        elif t < 6:
            items.append(g.work(p.id, g.GD_KIND_GATHER, mode, ptr=(b + C5_OUT_OFF, b, b + C5_IDX_OFF),
                                u64=(C5_N_IDX,), u32=(1,)))
            nbytes += 12 * C5_N_IDX
        else:
            items.append(g.work(p.id, g.GD_KIND_GEMM, mode, ptr=(b + 2 * n * n * 2, b, b + n * n * 2),
                                u64=(n, n, n), u32=(n, n, n)))
            flops += 2 * n ** 3
    return items, nbytes, flops


def c5_expected_violations(launches, world):
    """Check-mode violations C5 must count: 3 gather tenants x 671,089 planted
    indices (1 % of 2^26, synth.planted_count) x launches x GPUs."""
    import synth
    return 3 * synth.planted_count(0.01, C5_N_IDX) * launches * world


# ---------------------------------------------------------------------------
# the GPU arm
# ---------------------------------------------------------------------------

class Workload:
    def __init__(self, device: int):
        import torch
        from paper_2401_09290_b200 import devmem, guardian as g
        self.torch, self.g, self.devmem = torch, g, devmem
        self.device = device
        self.arena = g.Arena(device, ARENA)
        self.parts = [self.arena.partition_alloc(PART) for _ in range(TENANTS)]
        self.streams = [torch.cuda.Stream(device=device) for _ in range(TENANTS)]
        for t, p in enumerate(self.parts):
            gen = torch.Generator(device=f"cuda:{device}")
            gen.manual_seed(1000 * 2 + t)                              # seed = 1000*config + tenant
            devmem.view(p.base + OFF_SRC, COPY_BYTES // 4, torch.int32, device).random_(generator=gen)
            devmem.view(p.base + OFF_X, SAXPY_N, torch.float32, device).uniform_(-1.0, 1.0, generator=gen)
            devmem.view(p.base + OFF_Y, SAXPY_N, torch.float32, device).uniform_(-1.0, 1.0, generator=gen)
        torch.cuda.synchronize(device)

    def items(self, mode):
        return c2_items(self.g, self.parts, mode)

    def step(self, items):
        return self.arena.launcher_run(items, self.streams)

    def time_steps(self, mode, steps):
        """Shared start/stop events around `steps` launcher steps (makespan)."""
        torch = self.torch
        items = self.items(mode)
        root = torch.cuda.current_stream(self.device)
        start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ends = [torch.cuda.Event() for _ in self.streams]
        barrier()
        torch.cuda.synchronize(self.device)
        start.record(root)
        for s in self.streams:
            s.wait_event(start)
        for _ in range(steps):
            self.step(items)
        for s, e in zip(self.streams, ends):
            e.record(s)
            root.wait_event(e)
        stop.record(root)
        torch.cuda.synchronize(self.device)
        barrier()
        return start.elapsed_time(stop)                                # ms

    def solo_kernel_ms(self, mode, kind, reps):
        """Per-launch durations of one kernel launched back-to-back on one
        stream, CUDA events on that stream (the roofline's denominator)."""
        torch = self.torch
        p = self.parts[0]
        s = self.streams[0]
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(reps + 1)]
        with torch.cuda.stream(s):
            for _ in range(2):
                self._launch(kind, mode, p, s)
            evs[0].record(s)
            for i in range(reps):
                self._launch(kind, mode, p, s)
                evs[i + 1].record(s)
        torch.cuda.synchronize(self.device)
        return [evs[i].elapsed_time(evs[i + 1]) for i in range(reps)]

    def _launch(self, kind, mode, p, s):
        if kind == "copy":
            self.arena.copy(p.id, mode, p.base + OFF_DST, p.base + OFF_SRC, COPY_BYTES, stream=s)
        else:
            self.arena.saxpy(p.id, mode, ALPHA, p.base + OFF_X, p.base + OFF_Y, SAXPY_N, stream=s)

    def c5_setup(self, seed_base=5000):
        """C5 inputs: the gather tenants' indices (1 % planted out of the
        partition, synth.indices_with_oob) and the GEMM tenants' operands.
        Returns the planted count of one round."""
        import synth
        torch, devmem = self.torch, self.devmem
        n, planted = C5_GEMM_N, 0
        for t, p in enumerate(self.parts):
            b = p.base
            if 3 <= t < 6:
                idx, pos = synth.indices_with_oob(synth.rng_for(seed_base + t), C5_N_IDX, C5_TABLE_N, 0.01)
                devmem.view(b + C5_IDX_OFF, C5_N_IDX, torch.int32, self.device).copy_(torch.from_numpy(idx))
                planted += len(pos)
            elif t >= 6:
                gen = torch.Generator(device=f"cuda:{self.device}")
                gen.manual_seed(seed_base + t)
                for off in (0, n * n * 2):
                    devmem.view(b + off, n * n, torch.bfloat16, self.device).uniform_(-1, 1, generator=gen)
        torch.cuda.synchronize(self.device)
        return planted

    def c5(self, planted, launches=20, mode="check", policy="round_robin"):
        """BASELINE.json configs[4] on this GPU (c5_items), `launches`
        launches per tenant, issued by the launcher on 8 streams under
        `policy`.  Returns (makespan ms, bytes, flops, planted)."""
        torch = self.torch
        items, nbytes, flops = c5_items(self.g, self.parts, mode)
        queue = [it for it in items for _ in range(launches)]
        self.step(queue[:len(items)])                                     # warm-up round
        torch.cuda.synchronize(self.device)
        self.arena.stats_reset()
        root = torch.cuda.current_stream(self.device)
        start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        barrier()
        torch.cuda.synchronize(self.device)
        start.record(root)
        for s in self.streams:
            s.wait_event(start)
        self.arena.launcher_run(queue, self.streams, policy=policy)
        for s in self.streams:
            e = torch.cuda.Event()
            e.record(s)
            root.wait_event(e)
        stop.record(root)
        torch.cuda.synchronize(self.device)
        return start.elapsed_time(stop), nbytes * launches, flops * launches, planted * launches

    def kernel_table(self, reps=5, modes=ALL_MODES, per_access=False):
        """Solo launches of every kernel at its BASELINE size in `modes`,
        interleaved, CUDA events on one stream (after c5_setup(): tenant 3/4
        hold the C3 gather / scatter layout with 1 % OOB, tenant 6 the GEMM).
        per_access: every fenced mode with GD_FENCE_PER_ACCESS (the paper's
        instrumentation: no tile-level range test); the descriptor-fenced
        TMA kernels (GEMM, K5 v2) have no per-access fence and are left out.
        Returns {kernel: {mode: {"ms", "work", "unit"}}} (per GPU, medians)."""
        torch, parts = self.torch, self.parts
        n_idx, n = 1 << 26, 8192
        H = W = 32768
        p0, p3, p4, p5, p6 = parts[0], parts[3], parts[4], parts[5], parts[6]
        a = self.arena
        kern = {
            "copy_4GiB": (lambda m, s: a.copy(p0.id, m, p0.base + OFF_DST, p0.base + OFF_SRC, COPY_BYTES, stream=s),
                          BYTES_COPY, "GB/s"),
            "saxpy_2^30": (lambda m, s: a.saxpy(p0.id, m, ALPHA, p0.base + OFF_X, p0.base + OFF_Y, SAXPY_N, stream=s),
                           BYTES_SAXPY, "GB/s"),
            "gather_2^26_1pct_oob": (lambda m, s: a.gather(p3.id, m, p3.base + 2 * GiB + GiB // 4, p3.base,
                                                           p3.base + 2 * GiB, n_idx, stream=s), 12 * n_idx, "GB/s"),
            "scatter_2^26_1pct_oob": (lambda m, s: a.scatter(p4.id, m, p4.base, p4.base + 2 * GiB,
                                                             p4.base + 2 * GiB + GiB // 4, n_idx, stream=s),
                                      16 * n_idx, "GB/s"),
            "stencil_32768^2": (lambda m, s: a.stencil(p5.id, m, p5.base + 8 * GiB, p5.base + 4 * GiB, H, W, W,
                                                       0.5, 0.125, stream=s), 8 * (H - 2) * (W - 2), "GB/s"),
            "gather_rows_D32_1GiB": (lambda m, s: a.gather(p5.id, m, p5.base + 3 * GiB, p5.base,
                                                           p5.base + 2 * GiB + GiB // 2, GiB // 128, 32, stream=s),
                                     4 * (GiB // 128) + 2 * GiB, "GB/s"),       # 4 + 8 D bytes per row
        }
        if not per_access:
            kern["stencil_tma_32768^2"] = (lambda m, s: a.stencil_tma(p5.id, m, p5.base + 8 * GiB, p5.base + 4 * GiB,
                                                                      H, W, W, 0.5, 0.125, stream=s),
                                           8 * (H - 2) * (W - 2), "GB/s")
            kern["gemm_8192^3"] = (lambda m, s: a.gemm(p6.id, m, p6.base + 2 * n * n * 2, p6.base,
                                                       p6.base + n * n * 2, n, n, n, n, n, n, stream=s),
                                   2 * n ** 3, "TFLOP/s")
        s = self.streams[0]
        out = {}
        launch_mode = {m: (m + "+pa" if per_access and m != "none" else m) for m in modes}
        for name, (fn, work, unit) in kern.items():
            times = {m: [] for m in modes}
            with torch.cuda.stream(s):
                for m in modes:
                    fn(launch_mode[m], s)
                for r in range(reps):
                    for m in rotated(modes, r):
                        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                        e0.record(s)
                        fn(launch_mode[m], s)
                        e1.record(s)
                        e1.synchronize()
                        times[m].append(e0.elapsed_time(e1))
            out[name] = {m: {"ms": statistics.median(v), "ms_paper_mean": paper_mean(v), "work": work, "unit": unit}
                         for m, v in times.items()}
        return out

    def rows_setup(self):
        """Embedding-row gather input (kernel_table's gather_rows_D32): 2^23
        row indices uniform over the 2^24 rows of 128 B of tenant 5's first
        2 GiB, at 2.5 GiB (its stencil buffers start at 4 GiB)."""
        torch, p5 = self.torch, self.parts[5]
        gen = torch.Generator(device=f"cuda:{self.device}")
        gen.manual_seed(5105)
        self.devmem.view(p5.base, 1 << 29, torch.int32, self.device).random_(generator=gen)
        self.devmem.view(p5.base + 2 * GiB + GiB // 2, GiB // 128, torch.int32, self.device).random_(
            0, (1 << 29) // 32, generator=gen)
        H = W = 32768
        self.devmem.view(p5.base + 4 * GiB, H * W, torch.float32, self.device).uniform_(0, 1, generator=gen)
        torch.cuda.synchronize(self.device)

    def l2_table(self, reps=5, modes=ALL_MODES, per_access=False, batch=50):
        """The L2-resident regime (the
        fence's ALU cost least hidden): working sets below the 126 MB L2 on
        tenant 7 (offset 1 GiB), each mode's batch of `batch` back-to-back
        launches captured once into a CUDA graph and replayed between two
        events (per-launch mean), modes interleaved."""
        torch, devmem, a, p = self.torch, self.devmem, self.arena, self.parts[7]
        b = p.base + GiB
        gen = torch.Generator(device=f"cuda:{self.device}")
        gen.manual_seed(5207)
        devmem.view(b, 8 * MiB, torch.int32, self.device).random_(generator=gen)
        devmem.view(b + 128 * MiB, 8 * MiB, torch.float32, self.device).uniform_(-1, 1, generator=gen)
        devmem.view(b + 192 * MiB, 8 * MiB, torch.float32, self.device).uniform_(-1, 1, generator=gen)
        n = 1 << 22
        devmem.view(b + 256 * MiB, n, torch.int32, self.device).random_(0, n, generator=gen)
        H = W = 2048
        devmem.view(b + 384 * MiB, H * W, torch.float32, self.device).uniform_(0, 1, generator=gen)
        torch.cuda.synchronize(self.device)
        kern = {
            "copy_32MiB": (lambda m, s: a.copy(p.id, m, b + 64 * MiB, b, 32 * MiB, stream=s), 2 * 32 * MiB),
            "saxpy_2^23": (lambda m, s: a.saxpy(p.id, m, 1.0, b + 128 * MiB, b + 192 * MiB, 8 * MiB, stream=s),
                           12 * 8 * MiB),
            "gather_2^22_into_2^22": (lambda m, s: a.gather(p.id, m, b + 320 * MiB, b, b + 256 * MiB, n, stream=s),
                                      12 * n),
            "stencil_2048^2": (lambda m, s: a.stencil(p.id, m, b + 448 * MiB, b + 384 * MiB, H, W, W, 0.5, 0.125,
                                                      stream=s), 8 * (H - 2) * (W - 2)),
        }
        if not per_access:
            kern["stencil_tma_2048^2"] = (lambda m, s: a.stencil_tma(p.id, m, b + 448 * MiB, b + 384 * MiB, H, W, W,
                                                                     0.5, 0.125, stream=s), 8 * (H - 2) * (W - 2))
        launch_mode = {m: (m + "+pa" if per_access and m != "none" else m) for m in modes}
        s = self.streams[7]
        out = {}
        for name, (fn, work) in kern.items():
            graphs, times = {}, {m: [] for m in modes}
            with torch.cuda.stream(s):
                for m in modes:
                    for _ in range(3):
                        fn(launch_mode[m], s)
                s.synchronize()
                for m in modes:
                    gr = torch.cuda.CUDAGraph()
                    with torch.cuda.graph(gr, stream=s):
                        for _ in range(batch):
                            fn(launch_mode[m], s)
                    graphs[m] = gr
                for m in modes:
                    graphs[m].replay()
                for r in range(reps):
                    for m in rotated(modes, r):
                        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                        e0.record(s)
                        graphs[m].replay()
                        e1.record(s)
                        e1.synchronize()
                        times[m].append(e0.elapsed_time(e1) / batch)
            out[name] = {m: {"ms": statistics.median(v), "ms_paper_mean": paper_mean(v), "work": work, "unit": "GB/s"}
                         for m, v in times.items()}
            del graphs
        return out

    def sample_c2(self, k=1 << 16, seed=2999):
        """Seeded sample of every tenant's C2 buffers, read back now: saxpy
        element positions (x, y) and copy 16-byte units (src, dst)."""
        import numpy as np
        torch, devmem = self.torch, self.devmem
        rng = np.random.default_rng(seed)
        out = []
        for p in self.parts:
            e = torch.from_numpy(np.sort(rng.integers(0, SAXPY_N, k))).to(f"cuda:{self.device}")
            u = torch.from_numpy(np.sort(rng.integers(0, COPY_BYTES // 16, k))).to(f"cuda:{self.device}")
            x = devmem.view(p.base + OFF_X, SAXPY_N, torch.float32, self.device)[e].cpu().numpy()
            y = devmem.view(p.base + OFF_Y, SAXPY_N, torch.float32, self.device)[e].cpu().numpy()
            src = devmem.view(p.base + OFF_SRC, COPY_BYTES // 8, torch.int64, self.device).view(-1, 2)[u]
            dst = devmem.view(p.base + OFF_DST, COPY_BYTES // 8, torch.int64, self.device).view(-1, 2)[u]
            out.append({"x": x, "y": y, "src": src.cpu().numpy().view(np.uint8).reshape(-1),
                        "dst": dst.cpu().numpy().view(np.uint8).reshape(-1)})
        return out

    def e2e(self, mode, steps, warmup):
        """Through the public API with HOST buffers: every step copies each
        tenant's inputs host->device (checked transfers, gd_memcpy_h2d), runs
        the fenced step, and reads the outputs back (gd_memcpy_d2h)."""
        torch = self.torch
        host_in = torch.empty(COPY_BYTES, dtype=torch.uint8, pin_memory=True)
        host_out = torch.empty(COPY_BYTES, dtype=torch.uint8, pin_memory=True)
        host_in.random_(0, 256)
        items = self.items(mode)
        a = self.arena

        per_tenant = [[it for it in items if it.tenant == p.id] for p in self.parts]

        def one():
            # tenant-major issue, each tenant on its own stream: upload, its
            # fenced kernels (the launcher with that tenant's stream), download.
            # The host->device engine serves the uploads in issue order, so
            # tenant t's kernels and download overlap the uploads of tenants
            # t+1.. (measured: 55.6 GB/s each way, 99 GB/s both,
            # tools/pcie_probe.py)
            for t, p in enumerate(self.parts):
                s = self.streams[t]
                for off in (OFF_SRC, OFF_X, OFF_Y):
                    a.memcpy_h2d(p.id, p.base + off, host_in.data_ptr(), COPY_BYTES, stream=s)
                a.launcher_run(per_tenant[t], [s])
                for off in (OFF_DST, OFF_Y):
                    a.memcpy_d2h(p.id, host_out.data_ptr(), p.base + off, COPY_BYTES, stream=s)
            # no host sync between steps: each tenant's stream orders its next
            # step's uploads after this step's downloads, so consecutive steps
            # pipeline across the two copy directions

        for _ in range(warmup):
            one()
        torch.cuda.synchronize(self.device)
        barrier()
        torch.cuda.synchronize(self.device)
        t0 = time.perf_counter()
        for _ in range(steps):
            one()
        torch.cuda.synchronize(self.device)
        el = time.perf_counter() - t0
        el = allreduce([el])[0]
        barrier()
        return el / steps, 3 * COPY_BYTES * TENANTS, 2 * COPY_BYTES * TENANTS


def ncu_traffic(kernel_tag: str):
    """DRAM bytes per launch and ncu's DRAM throughput (% of the theoretical
    peak) of `kernel_tag`, from the committed ncu --set full capture
    (profiles/ncu_traffic.json, written by tools/ncu_summary.py)."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if not os.path.exists(p):
        return None, None, None
    with open(p) as f:
        d = json.load(f)
    v = d.get(kernel_tag)
    pct = d.get(kernel_tag + ":dram_pct")
    return (v if isinstance(v, (int, float)) else None, pct if isinstance(pct, (int, float)) else None,
            d.get("_source"))


def reduce_table(table, world, modes):
    """Max time over ranks per kernel and mode; rate = world x work / time;
    overhead against the unfenced twin of the same table."""
    for row in table.values():
        for m in list(row):
            t, tp = allreduce([row[m]["ms"], row[m]["ms_paper_mean"]])
            u = row[m]["unit"]
            row[m] = {"ms": round(t, 5), "ms_paper_mean": round(tp, 5),
                      u: round(world * row[m]["work"] / (t / 1e3) / (1e9 if u == "GB/s" else 1e12), 1)}
        for m in modes:
            if m != "none":
                row[m]["overhead_pct"] = round(100 * (row[m]["ms"] / row["none"]["ms"] - 1), 2)
    return table


def run_gpu(args):
    import torch
    world, rank, local = dist_init()
    torch.cuda.set_device(local)
    hbm, bf16, bf16s, peak_src = peaks()
    w = Workload(local)

    # the clock sampler runs from the warm-up through the timed region (its
    # samples are 50 ms apart; the timed region alone is a few hundred ms)
    with Clocks(local) as clk:
        for _ in range(args.warmup):
            w.step(w.items(args.mode))
        torch.cuda.synchronize(local)

        # ---- the contract's timed region: exactly K steps, max over ranks ----
        pre = w.sample_c2()                               # parity sample of the inputs (not timed)
        ms = w.time_steps(args.mode, args.steps)
        post = w.sample_c2()                              # ... and of the outputs of the K timed steps
    ms = allreduce([ms])[0]
    ms_per_step = ms / args.steps
    value = world * STEP_BYTES_PER_GPU / (ms_per_step / 1e3) / 1e9

    # ---- overhead vs the unfenced twin: every mode, interleaved ----
    modes = ALL_MODES
    per_mode = {m: [] for m in modes}
    for r in range(args.reps):
        for m in rotated(modes, r):
            per_mode[m].append(allreduce([w.time_steps(m, args.steps)])[0] / args.steps)
    med = {m: statistics.median(v) for m, v in per_mode.items()}
    modes_gbs = {m: round(world * STEP_BYTES_PER_GPU / (med[m] / 1e3) / 1e9, 1) for m in med}
    overhead = {m: round(100.0 * (med[m] / med["none"] - 1.0), 2) for m in modes[1:]}

    # ---- roofline of the dominant kernel (saxpy: 12 B/element) ----
    solo = {}
    for kind, nbytes in (("saxpy", BYTES_SAXPY), ("copy", BYTES_COPY)):
        for m in ("none", args.mode):
            d = w.solo_kernel_ms(m, kind, args.steps)
            solo[(kind, m)] = (statistics.mean(d), nbytes)
    sx_ms, sx_bytes = solo[("saxpy", args.mode)]
    achieved = sx_bytes / (sx_ms / 1e3) / 1e9
    mode_id = ALL_MODES.index(args.mode)
    if args.mode == "mask" and ncu_traffic("k_saxpy<6>")[0] is not None:
        mode_id = 6          # mask on a >= 4 GiB partition launches k_saxpy<kMaskBig> (fence_desc.h)
    traffic, dram_pct, traffic_src = ncu_traffic(f"k_saxpy<{mode_id}>")
    roofline = {"bound": "hbm", "achieved": round(achieved, 1), "peak": hbm, "unit": "GB/s",
                "frac": round(achieved / hbm, 4), "traffic": traffic,
                "traffic_source": ("committed ncu --set full capture of this kernel (profiles/ncu_traffic.json"
                                   + (f", {traffic_src}" if traffic_src else "") + "), not measured in this run"),
                "ncu_dram_throughput_pct_of_theoretical": dram_pct,
                "kernel": f"k_saxpy<{args.mode}>", "peak_source": f"{peak_src} copy bandwidth (MEASURED_PEAKS.json)",
                "bytes_per_launch": sx_bytes, "avg_launch_ms": round(sx_ms, 4),
                "share_of_step": round(TENANTS * sx_ms / (TENANTS * (sx_ms + solo[("copy", args.mode)][0])), 3),
                # the measured peak is torch's copy_, which this kernel beats; against
                # the theoretical 8.18 TB/s (8192-bit bus x 2 x 3996 MHz, ncu's
                # denominator) and the HGX nominal 7.7 TB/s the same launch is:
                "theoretical_peak": 8184.0, "frac_of_theoretical": round(achieved / 8184.0, 4),
                "nominal_peak": 7700.0, "frac_of_nominal": round(achieved / 7700.0, 4)}
    kernels = {f"{k}/{m}": {"ms": round(t, 4), "GB/s": round(b / (t / 1e3) / 1e9, 1)}
               for (k, m), (t, b) in solo.items()}

    # ---- end to end through the C ABI with host buffers ----
    e2e = None
    if not args.no_e2e:
        s_per_step, h2d, d2h = w.e2e(args.mode, args.e2e_steps, 1)
        e2e = {"value": round(world * STEP_BYTES_PER_GPU / s_per_step / 1e9, 2), "unit": "GB/s",
               "h2d_bytes_per_step": world * h2d, "d2h_bytes_per_step": world * d2h,
               "steps": args.e2e_steps, "note": "pinned host buffers, checked gd_memcpy_h2d/d2h, tenant-major pipelined issue; "
                       "bound by the uploads: 103 GB per step at the box's measured 55.6 GB/s host->device "
                       "(profiles/r01_pcie_probe.txt) caps e2e at ~92.7 GB/s"}

    # ---- C5: mixed tenants (copy / gather 1 % OOB / GEMM) in check mode ----
    c5 = None
    c5_expected = 0
    if not args.no_c5:
        # headline: the paper's launcher (round robin, free-running tenant
        # streams); beside it the interference-aware
        # memory-lane policy (include/guardian.h gd_policy).  Round robin runs
        # last, so the violation check below reads its counters.
        planted = w.c5_setup()
        by_policy = {}
        for pol in ("memory_lane", "round_robin"):
            c5_ms, c5_bytes, c5_flops, c5_planted = w.c5(planted, launches=args.c5_launches, policy=pol)
            by_policy[pol] = allreduce([c5_ms])[0]
        c5_ms_max = by_policy["round_robin"]
        c5_expected = int(allreduce([float(c5_planted)], op="sum")[0])
        assert c5_expected == c5_expected_violations(args.c5_launches, world)
        c5 = {"makespan_ms": round(c5_ms_max, 3), "policy": "round_robin",
              "launches_per_tenant": args.c5_launches, "mode": "check",
              "memory_GBps": round(world * c5_bytes / (c5_ms_max / 1e3) / 1e9, 1),
              "gemm_TFLOPs": round(world * c5_flops / (c5_ms_max / 1e3) / 1e12, 1),
              "memory_lane": {"makespan_ms": round(by_policy["memory_lane"], 3),
                              "memory_GBps": round(world * c5_bytes / (by_policy["memory_lane"] / 1e3) / 1e9, 1),
                              "gemm_TFLOPs": round(world * c5_flops / (by_policy["memory_lane"] / 1e3) / 1e12, 1)},
              "tenants": "t0-2 copy 4 GiB, t3-5 gather 2^26 (1% OOB), t6-7 GEMM 8192^3 bf16"}

    # ---- statistics reduced over GPUs with NCCL (the one collective) ----
    from paper_2401_09290_b200 import dist as gdist
    per = {rank * TENANTS + t: w.arena.stats(p.id) for t, p in enumerate(w.parts)}
    red_t, span = gdist.allreduce_stats(per, ms, world * TENANTS)
    red = [sum(d[f] for d in red_t.values()) for f in ("violations", "launches", "bytes")]
    if c5 is not None:
        c5["violations_allreduced"] = int(red[0])
        c5["violations_expected"] = c5_expected
        c5["violations_expected_formula"] = f"3 x 671,089 x {args.c5_launches} launches x {world} GPU(s)"
        c5["violations_exact"] = int(red[0]) == c5_expected

    # ---- every kernel x every mode at the BASELINE sizes,
    #      hoisted (default) and per access; the L2-resident regime ----
    table = table_pa = l2 = l2_pa = None
    tables_clocks = {}
    if not args.no_c5:
        w.rows_setup()
        # the SM clock during each table (nvidia-smi, 50 ms samples): late in a
        # long run the power cap lowers it, which slows the ALU-heavier
        # per-access variants more than their memory-bound twins
        with Clocks(local) as ck:
            table = reduce_table(w.kernel_table(reps=args.table_reps), world, ALL_MODES)
        tables_clocks["kernels_all_modes"] = ck.summary()
        with Clocks(local) as ck:
            table_pa = reduce_table(w.kernel_table(reps=args.table_reps, per_access=True), world, ALL_MODES)
        tables_clocks["kernels_all_modes_per_access"] = ck.summary()
        with Clocks(local) as ck:
            l2 = reduce_table(w.l2_table(reps=args.table_reps), world, ALL_MODES)
        tables_clocks["l2_resident"] = ck.summary()
        with Clocks(local) as ck:
            l2_pa = reduce_table(w.l2_table(reps=args.table_reps, per_access=True), world, ALL_MODES)
        tables_clocks["l2_resident_per_access"] = ck.summary()

    # ---- parity of the timed steps (cpu_baseline leg: the oracle on the host
    #      re-computes the sampled outputs; every rank checks its tenants) ----
    par = oracle_parity(pre, post, args.steps, args.mode)
    bad = int(allreduce([float(par["mismatches"])], op="sum")[0])
    parity = {"status": "ok" if bad == 0 else "FAIL", "mismatches": bad,
              "checked": int(allreduce([float(par["checked"])], op="sum")[0]),
              "sample": par["sample"]}

    cpu = None
    if rank == 0 and not args.no_cpu:
        cpu = cpu_baseline(seconds=args.cpu_seconds)
        cpu["by_config"] = cpu_by_config("mask", host_threads(), table)

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 1), "unit": "GB/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms_per_step, 3), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (torch.Generator seeded 1000*2+tenant: random bytes, U[-1,1) fp32)",
            "config": gpu_config(args.mode, world),
            "per_gpu_GBps": round(value / world, 1),
            "frac_of_hbm_peak": round(value / world / hbm, 4),
            "parity": parity["status"], "parity_detail": parity,
            "modes_GBps": modes_gbs, "overhead_pct_vs_unfenced": overhead,
            "roofline": roofline, "kernels_solo": kernels,
            "e2e": e2e, "gpu_launches": args.steps * 2 * TENANTS,
            "clocks": clk.summary(),
            "stats_allreduced": {"violations": int(red[0]), "launches": int(red[1]), "bytes": int(red[2])},
            "multi_tenant_c5": c5,
            "kernels_all_modes": table,
            "kernels_all_modes_per_access": table_pa,
            "l2_resident": l2,
            "l2_resident_per_access": l2_pa,
            "tables_clocks": tables_clocks,
            "cpu_baseline": cpu,
        }
        emit(line)
    w.arena.close()


def run_dry(args):
    """--dry-run: the rank plumbing of run_gpu on CPU -- gloo process group,
    one VIRTUAL arena per rank (gd_arena_wrap with device -1: the partition
    manager and the launcher's validation run, nothing launches), the C2 and
    C5 items validated, max-over-ranks timing and the stats all_reduce.  The
    per-rank counters are the ones C5 plants (3 gather tenants x 671,089 x
    launches); the timing is a placeholder.  Prints ONE JSON line on rank 0."""
    from paper_2401_09290_b200 import dist as gdist, guardian as g
    world, rank, local = dist_init("gloo")
    arena = g.Arena.wrap(-1, ARENA * (rank + 1), ARENA)                # size-aligned fake VA per rank
    parts = [arena.partition_alloc(PART) for _ in range(TENANTS)]
    assert [p.base for p in parts] == [arena.base + t * PART for t in range(TENANTS)]
    valid = 0
    for items in (c2_items(g, parts, args.mode), c5_items(g, parts, "check")[0]):
        try:
            arena.launcher_run(items, [None] * TENANTS)
        except g.GuardianError as e:                                  # validated: no device to run on
            assert e.status == g.GD_ERR_UNSUPPORTED, e
        valid += len(items)
    ms = allreduce([10.0 + rank])[0]                                   # placeholder, max over ranks
    per = {}
    for t, p in enumerate(parts):
        planted = 671089 if 3 <= t < 6 else 0
        per[rank * TENANTS + t] = {"violations": planted * args.c5_launches, "launches": args.c5_launches,
                                   "bytes": 0, "flops": 0}
    red_t, span = gdist.allreduce_stats(per, ms, world * TENANTS)
    red = [sum(d[f] for d in red_t.values()) for f in ("violations", "launches", "bytes")]
    expected = c5_expected_violations(args.c5_launches, world)
    if rank == 0:
        emit({"metric": METRIC, "value": None, "unit": "GB/s", "n_gpus": world, "steps": args.steps,
              "warmup": args.warmup, "ms_per_step": None, "higher_is_better": True, "scaling": "weak",
              "dry_run": True, "items_validated_per_rank": valid, "makespan_ms_max": span,
              "stats_allreduced": {"violations": int(red[0]), "launches": int(red[1]), "bytes": int(red[2])},
              "multi_tenant_c5": {"violations_allreduced": int(red[0]), "violations_expected": expected,
                                  "violations_exact": int(red[0]) == expected}})
    arena.close()


def oracle_parity(pre, post, steps, mode):
    """Part of the cpu_baseline leg (the oracle on the host cores, after all
    GPU timing): re-compute the sampled outputs of the K timed steps.  Every
    timed step applied, per tenant, y <- fmaf(a, x, y) (saxpy) and dst <- src
    (copy) once, so on the sample y after the timed region must equal K
    oracle saxpy passes over (x, y before it), bit for bit, and dst the
    oracle's copy of src."""
    import numpy as np
    import oracle
    bad = checked = 0
    base, size = 0x7E0000000000, 1 << 24
    for a, b in zip(pre, post):
        k = len(a["x"])
        m = oracle.Mem(base, size)
        m.write(base, a["x"])
        m.write(base + 4 * k, a["y"])
        m.write(base + 8 * k, b["src"])
        for _ in range(steps):
            oracle.saxpy(m, base, size, mode, ALPHA, base, base + 4 * k, k)
        oracle.copy(m, base, size, mode, base + 8 * k + 16 * k, base + 8 * k, 16 * k)
        bad += int(np.count_nonzero(m.view(base + 4 * k, np.uint32, k) != b["y"].view(np.uint32)))
        bad += int(np.count_nonzero(m.view(base + 24 * k, np.uint8, 16 * k) != b["dst"]))
        bad += int(np.count_nonzero(a["src"] != b["src"]))            # the copy source is never written
        checked += k + 16 * k
    k = len(pre[0]["x"]) if pre else 0
    return {"mismatches": bad, "checked": checked,
            "sample": f"per tenant {k} seeded saxpy elements (y after the {steps} timed steps vs {steps} oracle "
                      f"passes) and {k} copy 16-byte units, bit-exact"}


# ---------------------------------------------------------------------------
# the CPU oracle (cpu_baseline leg and --impl reference)
# ---------------------------------------------------------------------------

SAMPLE_COPY = 64 << 20            # bytes per tenant sample
SAMPLE_SAXPY = 16 << 20           # elements per tenant sample


class OracleSample:
    """A bounded sample of the C2 workload simulated by the CPU oracle: per
    tenant a 256 MiB slice of its partition holding a 64 MiB copy and a
    2^24-element SAXPY (same kernels, same fence, same mode)."""

    def __init__(self, threads: int, mode: str):
        import numpy as np
        import oracle
        import synth
        self.oracle, self.mode = oracle, mode
        self.threads = threads
        self.mems = []
        for t in range(threads):
            base = 0x7F0000000000 + t * PART
            m = oracle.Mem(base, 4 * SAMPLE_COPY)
            rng = synth.rng_for(1000 * 2 + t)
            m.buf[:SAMPLE_COPY] = synth.random_bytes(rng, SAMPLE_COPY)
            m.write(base + 2 * SAMPLE_COPY, synth.uniform_f32(rng, SAMPLE_SAXPY))
            m.write(base + 3 * SAMPLE_COPY, synth.uniform_f32(rng, SAMPLE_SAXPY))
            self.mems.append((m, base))
        self.bytes_per_pass = threads * (2 * SAMPLE_COPY + 12 * SAMPLE_SAXPY)

    def one(self, i):
        m, base = self.mems[i]
        o = self.oracle
        o.copy(m, base, PART, self.mode, base + SAMPLE_COPY, base, SAMPLE_COPY)
        o.saxpy(m, base, PART, self.mode, ALPHA, base + 2 * SAMPLE_COPY, base + 3 * SAMPLE_COPY, SAMPLE_SAXPY)

    def run_pass(self):
        from concurrent.futures import ThreadPoolExecutor
        with ThreadPoolExecutor(self.threads) as ex:
            list(ex.map(self.one, range(self.threads)))


def host_threads():
    try:
        n = len(os.sched_getaffinity(0))
    except AttributeError:
        n = os.cpu_count() or 1
    return max(1, min(TENANTS, n))


def cpu_baseline(seconds: float = 12.0, mode: str = "mask"):
    th = host_threads()
    s = OracleSample(th, mode)
    t0 = time.perf_counter()
    passes = 0
    while True:
        s.run_pass()
        passes += 1
        if time.perf_counter() - t0 >= seconds:
            break
    el = time.perf_counter() - t0
    return {"value": round(passes * s.bytes_per_pass / el / 1e9, 3), "unit": "GB/s", "cores": th, "kind": "oracle",
            "sample": f"{passes} pass(es) x {th} tenants x (64 MiB copy + 2^24-element saxpy), mode={mode}, "
                      f"{el:.1f} s"}


# ---------------------------------------------------------------------------
# cpu_baseline leg, per BASELINE config (SURVEY.md §8(d) "Oracle timing"):
# the oracle as it stands on a bounded sample of every config, one tenant per
# host thread, and the GPU/oracle ratio against this run's own kernel table.
# ---------------------------------------------------------------------------
OBASE = 0x7F0000000000


def _oimports():
    import numpy as np
    import oracle
    import synth
    return np, oracle, synth


def _otimed(fn, th):
    from concurrent.futures import ThreadPoolExecutor
    t0 = time.perf_counter()
    with ThreadPoolExecutor(th) as ex:
        list(ex.map(fn, range(th)))
    return time.perf_counter() - t0


def _ocfg_c1(mode):
    np, oracle, synth = _oimports()
    g = synth.toy_gather()
    m = oracle.Mem(OBASE, synth.C1_ARENA)
    for t in range(synth.C1_TENANTS):
        b = OBASE + t * synth.C1_PART
        m.write(b + synth.C1_TABLE_OFF, g.tables[t])
        m.write(b + synth.C1_IDX_OFF, g.idx[t])
    t0 = time.perf_counter()
    for t in range(synth.C1_TENANTS):
        b = OBASE + t * synth.C1_PART
        oracle.gather(m, b, synth.C1_PART, mode, b + synth.C1_OUT_OFF, b + synth.C1_TABLE_OFF, b + synth.C1_IDX_OFF,
                      synth.C1_N, 1)
    el = time.perf_counter() - t0
    n = synth.C1_TENANTS * synth.C1_N
    return {"sample": f"whole C1: {n} indices, 4 tenants, one thread", "seconds": round(el, 3),
            "GB/s": round(12 * n / el / 1e9, 4), "cores": 1}


def _ocfg_c2(mode, th):
    np, oracle, synth = _oimports()
    cp, sx = 64 * MiB, 1 << 24
    mems = []
    for t in range(th):
        b = OBASE + t * PART
        m = oracle.Mem(b, 4 * cp)
        rng = synth.rng_for(2000 + t)
        m.buf[:cp] = synth.random_bytes(rng, cp)
        m.write(b + 2 * cp, synth.uniform_f32(rng, sx))
        m.write(b + 3 * cp, synth.uniform_f32(rng, sx))
        mems.append((m, b))

    def one(i):
        m, b = mems[i]
        oracle.copy(m, b, PART, mode, b + cp, b, cp)
        oracle.saxpy(m, b, PART, mode, 1.5, b + 2 * cp, b + 3 * cp, sx)
    el = _otimed(one, th)
    return {"sample": f"{th} tenants x (64 MiB copy + 2^24-element saxpy)", "seconds": round(el, 3),
            "GB/s": round(th * (2 * cp + 12 * sx) / el / 1e9, 3), "cores": th}


def _ocfg_c3(mode, th):
    np, oracle, synth = _oimports()
    T, n = 1 << 26, 1 << 22
    mems = []
    for t in range(th):
        b = OBASE + t * PART
        m = oracle.Mem(b, 4 * T + 8 * n)
        rng = synth.rng_for(3000 + t)
        m.write(b, rng.integers(0, 2**32, T, dtype=np.uint64).astype(np.uint32))
        j = rng.integers(0, T, n, dtype=np.int64)
        pos = synth.planted_positions(rng, n, synth.planted_count(0.01, n))
        j[pos] = rng.integers(-2**31, 0, len(pos))
        m.write(b + 4 * T, j.astype(np.int32))
        mems.append((m, b))

    def one(i):
        m, b = mems[i]
        oracle.gather(m, b, PART, mode, b + 4 * T + 4 * n, b, b + 4 * T, n, 1)
    el = _otimed(one, th)
    return {"sample": f"{th} tenants x 2^22 indices into a 2^26-word table, 1 % planted OOB",
            "seconds": round(el, 3), "GB/s": round(th * 12 * n / el / 1e9, 3), "cores": th}


def _ocfg_c4_gemm(mode):
    np, oracle, synth = _oimports()
    n, rows = 8192, 16
    b = OBASE
    m = oracle.Mem(b, 3 * n * n * 2)
    rng = synth.rng_for(4006)
    m.write(b, synth.bf16_bits_uniform(rng, n * n))
    m.write(b + n * n * 2, synth.bf16_bits_uniform(rng, n * n))
    sel = np.sort(rng.permutation(n)[:rows]).astype(np.uint32)
    t0 = time.perf_counter()
    oracle.gemm(m, b, PART, mode, b + 2 * n * n * 2, b, b + n * n * 2, n, n, n, n, n, n, rows=sel)
    el = time.perf_counter() - t0
    return {"sample": f"{rows} seeded full rows of C at 8192^3, one thread", "seconds": round(el, 3),
            "TFLOP/s": round(2 * rows * n * n / el / 1e12, 6), "cores": 1}


def _ocfg_c4_stencil(mode, th):
    np, oracle, synth = _oimports()
    H = W = 2048
    mems = []
    for t in range(th):
        b = OBASE + t * PART
        m = oracle.Mem(b, 8 * H * W)
        m.write(b, synth.uniform_f32(synth.rng_for(4100 + t), H * W, 0.0, 1.0))
        mems.append((m, b))

    def one(i):
        m, b = mems[i]
        oracle.stencil(m, b, PART, mode, b + 4 * H * W, b, H, W, W, 0.5, 0.125)
    el = _otimed(one, th)
    return {"sample": f"{th} tenants x 2048^2 stencil", "seconds": round(el, 3),
            "GB/s": round(th * 8 * (H - 2) * (W - 2) / el / 1e9, 3), "cores": th}



def cpu_by_config(mode, th, table=None):
    out = {"C1_toy_gather": _ocfg_c1(mode), "C2_copy_saxpy": _ocfg_c2(mode, th), "C3_gather": _ocfg_c3(mode, th),
           "C4_gemm": _ocfg_c4_gemm(mode), "C4_stencil": _ocfg_c4_stencil(mode, th)}
    if table:
        pick = {"C2_copy_saxpy": (("copy_4GiB", "saxpy_2^30"), "GB/s"), "C3_gather": (("gather_2^26_1pct_oob",), "GB/s"),
                "C4_gemm": (("gemm_8192^3",), "TFLOP/s"), "C4_stencil": (("stencil_32768^2",), "GB/s")}
        for k, (names, unit) in pick.items():
            vals = [table[n][mode][unit] for n in names if n in table and mode in table[n]]
            if vals:
                gpu = sum(vals) / len(vals)
                out[k]["gpu"] = gpu
                out[k]["gpu_over_oracle"] = round(gpu / out[k][unit], 1)
    return out


def run_reference(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    th = host_threads()
    s = OracleSample(th, args.mode)
    for _ in range(args.warmup):
        s.run_pass()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        s.run_pass()
    el = time.perf_counter() - t0
    value = args.steps * s.bytes_per_pass / el / 1e9
    line = {
        "metric": METRIC, "value": round(value, 3), "unit": "GB/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(1e3 * el / args.steps, 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (NumPy PCG64 seeded 1000*2+tenant)",
        # the config is our arm's, key for key (the contract: the reference arm
        # runs on our arm's config, each step a bounded sample of it); what a
        # step really runs is stated beside it, in sample_run
        "config": gpu_config(args.mode, world),
        "sample_run": {"tenants": th, "copy_bytes_per_tenant": SAMPLE_COPY, "saxpy_n_per_tenant": SAMPLE_SAXPY,
                       "parallelism": "host threads, one tenant per thread",
                       "note": "each step is a bounded sample of the config's C2 workload: the same kernels, "
                               "fence and mode over 64 MiB copies and 2^24-element saxpys per tenant "
                               "(the value is GB/s of algorithmic bytes, comparable across sizes)"},
        "impl": "reference",
        "cpu_baseline": {"value": round(value, 3), "unit": "GB/s", "cores": th, "kind": "oracle",
                         "sample": f"per step {th} tenants x (64 MiB copy + 2^24-element saxpy) of the C2 workload"},
        "e2e": {"value": round(value, 3), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--mode", default="mask", choices=list(ALL_MODES))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--reps", type=int, default=6, help="interleaved repetitions of the six modes (rotated order)")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-c5", action="store_true", help="skip the mixed multi-tenant (configs[4]) measurement")
    ap.add_argument("--c5-launches", type=int, default=20)
    ap.add_argument("--table-reps", type=int, default=6, help="a multiple of 6: every mode once in every position")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--dry-run", action="store_true",
                    help="the rank plumbing on CPU: gloo, virtual arenas, validation only, no kernels")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
        return 0
    world_env = os.environ.get("WORLD_SIZE")
    if world_env is None and args.gpus > 1:
        return spawn_ranks(args)                       # N ranks under torch.distributed.run
    if world_env is not None and int(world_env) != args.gpus:
        sys.stderr.write(f"bench.py: WORLD_SIZE={world_env} but --gpus {args.gpus}\n")
        return 2
    quiet_stdout()
    if args.dry_run:
        run_dry(args)
    else:
        run_gpu(args)
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized():
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
