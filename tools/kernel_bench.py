"""Per-kernel throughput at the BASELINE.json sizes, fenced vs unfenced.

For every kernel (C2 copy/saxpy, C3 gather/scatter at 0/1/10 % OOB, C4 stencil
32768^2 and GEMM 8192^3) the three modes are timed interleaved (none, mask,
check) with CUDA events on the launching stream, R repetitions after warm-up;
reports the median, the paper-style mean of 10 without min/max,
GB/s (TFLOP/s), fraction of the measured peak and overhead vs the unfenced
twin.  Check-mode violation counts are verified against the planted counts.

  python tools/kernel_bench.py [--reps 12] [--only gather,gemm] > out.json
"""
import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2401_09290_b200 import devmem, guardian as g  # noqa: E402

GiB = 1 << 30
PART = 1 << 34


def peaks():
    d = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    return d["hbm_gbs"], d["bf16_tflops"], d["bf16_tflops_sustained"]


def paper_mean(xs):
    xs = sorted(xs)
    core = xs[1:-1] if len(xs) > 2 else xs
    return statistics.mean(core)


MODES = ["none", "mask", "check", "modulo"]          # --modes


def time_modes(launch, reps, warm=3, extra=None):
    """launch(mode, stream) -> None; interleaved none/mask/check (+ extra
    reference launches {name: fn(stream)} timed in the same rotation)."""
    s = torch.cuda.Stream()
    res = {m: [] for m in MODES}
    extra = extra or {}
    res.update({k: [] for k in extra})

    def go(m):
        if m in extra:
            extra[m](s)
        else:
            launch(m, s)

    with torch.cuda.stream(s):
        for m in res:
            for _ in range(warm):
                go(m)
        order = list(res)
        for r in range(reps):
            for m in order[r % len(order):] + order[:r % len(order)]:     # rotated: every position once
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(s)
                go(m)
                b.record(s)
                b.synchronize()
                res[m].append(a.elapsed_time(b))
    return res


def time_modes_batched(launch, reps, batch=50, warm=3):
    """L2-resident regime: kernels of a few microseconds are timed as a batch
    of back-to-back launches between two events (per-launch mean).  Each
    mode's batch is captured once into a CUDA graph and replayed, so the
    host cost of a launch through the binding (several microseconds of
    Python + C ABI) cannot hide the kernel time."""
    s = torch.cuda.Stream()
    res = {m: [] for m in MODES}
    graphs = {}
    with torch.cuda.stream(s):
        for m in res:
            for _ in range(warm):
                launch(m, s)
        s.synchronize()
        for m in res:
            gr = torch.cuda.CUDAGraph()
            with torch.cuda.graph(gr, stream=s):
                for _ in range(batch):
                    launch(m, s)
            graphs[m] = gr
        for m in res:
            graphs[m].replay()
        order = list(res)
        for r in range(reps):
            for m in order[r % len(order):] + order[:r % len(order)]:     # rotated: every position once
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(s)
                graphs[m].replay()
                b.record(s)
                b.synchronize()
                res[m].append(a.elapsed_time(b) / batch)
    return res


def summarize(name, res, work, unit, peak):
    out = {}
    for m, xs in res.items():
        med = statistics.median(xs)
        rate = work / (med / 1e3) / (1e9 if unit == "GB/s" else 1e12)
        out[m] = {"ms_median": round(med, 6), "ms_paper_mean": round(paper_mean(xs), 6), unit: round(rate, 1),
                  "frac_of_peak": round(rate / peak, 4)}
    base = statistics.median(res["none"])
    for m in (m for m in MODES if m != "none"):
        out[m]["overhead_pct"] = round(100 * (statistics.median(res[m]) / base - 1), 2)
    print(f"{name:28s} " + "  ".join(f"{m}: {out[m][unit]:8.1f} {unit}" + (f" ({out[m]['overhead_pct']:+.2f}%)"
                                                                           if m != 'none' else '')
                                     for m in out), file=sys.stderr)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=12)
    ap.add_argument("--only", default="")
    ap.add_argument("--modes", default=",".join(MODES),
                    help="fence modes timed interleaved (none first): none,mask,check,modulo,maskcount,clamp")
    args = ap.parse_args()
    MODES[:] = args.modes.split(",")
    assert MODES[0] == "none", "none (the unfenced twin) must come first"
    only = set(args.only.split(",")) if args.only else None
    hbm, bf16, bf16s = peaks()
    torch.cuda.set_device(0)
    # KB_SLOTS=8: an 8 x 16 GiB arena (the bench's layout), the last partition
    # timed (placement probe); default: a victim and the timed partition
    slots = int(os.environ.get("KB_SLOTS", "2"))
    arena = g.Arena(0, slots * PART)
    parts = [arena.partition_alloc(PART) for _ in range(slots)]
    victim, p = parts[0], parts[-1]
    b = p.base
    gen = torch.Generator(device="cuda:0")
    gen.manual_seed(2001)
    results = {"peaks": {"hbm_gbs": hbm, "bf16_tflops": bf16, "bf16_tflops_sustained": bf16s},
               "device": torch.cuda.get_device_name(0)}

    def want(k):
        return only is None or k in only

    if want("copy") or want("saxpy"):
        devmem.view(b, GiB, torch.int32).random_(generator=gen)
        devmem.view(b + 8 * GiB, 1 << 30, torch.float32).uniform_(-1, 1, generator=gen)
        devmem.view(b + 12 * GiB, 1 << 30, torch.float32).uniform_(-1, 1, generator=gen)
    if want("copy"):
        r = time_modes(lambda m, s: arena.copy(p.id, m, b + 4 * GiB, b, 4 * GiB, stream=s), args.reps)
        results["copy_4GiB"] = summarize("copy 4 GiB", r, 2 * 4 * GiB, "GB/s", hbm)
    if want("saxpy"):
        r = time_modes(lambda m, s: arena.saxpy(p.id, m, 1.5, b + 8 * GiB, b + 12 * GiB, 1 << 30, stream=s),
                       args.reps)
        results["saxpy_2^30"] = summarize("saxpy 2^30", r, 12 * (1 << 30), "GB/s", hbm)

    if want("gather") or want("scatter"):
        # C3 layout: table 2^29 u32 @0, idx 2^26 @2 GiB, out/src @2.25 GiB, pattern [2.5 GiB, 16 GiB)
        n, T = 1 << 26, 1 << 29
        devmem.view(b, T, torch.int32).random_(generator=gen)
        devmem.view(b + 2 * GiB + GiB // 4, n, torch.int32).random_(generator=gen)
        arena.fill(p.id, 1, 2 * GiB + GiB // 2, PART - 2 * GiB - GiB // 2)
        for frac in (0.0, 0.01, 0.1):
            rng = synth.rng_for(3000 + int(frac * 100))
            idx, pos = synth.indices_with_oob(rng, n, T, frac)
            devmem.view(b + 2 * GiB, n, torch.int32).copy_(torch.from_numpy(idx))
            torch.cuda.synchronize()
            if want("gather"):
                arena.stats_reset()
                arena.gather(p.id, "check", b + 2 * GiB + GiB // 4, b, b + 2 * GiB, n)
                v = arena.stats(p.id)["violations"]
                assert v == len(pos), (v, len(pos))
                r = time_modes(lambda m, s: arena.gather(p.id, m, b + 2 * GiB + GiB // 4, b, b + 2 * GiB, n, stream=s),
                               args.reps)
                res = summarize(f"gather 2^26 oob={frac}", r, 12 * n, "GB/s", hbm)
                res["violations_check"] = v
                results[f"gather_oob{frac}"] = res
            if want("scatter") and frac in (0.0, 0.01):
                arena.stats_reset()
                arena.scatter(p.id, "check", b, b + 2 * GiB, b + 2 * GiB + GiB // 4, n)
                v = arena.stats(p.id)["violations"]
                assert v == len(pos), (v, len(pos))
                r = time_modes(lambda m, s: arena.scatter(p.id, m, b, b + 2 * GiB, b + 2 * GiB + GiB // 4, n,
                                                          stream=s), args.reps)
                res = summarize(f"scatter 2^26 oob={frac}", r, 16 * n, "GB/s", hbm)
                res["violations_check"] = v
                results[f"scatter_oob{frac}"] = res

    if want("gatherrows"):
        # embedding rows: 2^29 u32 table viewed as rows of D words, indices into the row count
        T = 1 << 29
        devmem.view(b, T, torch.int32).random_(generator=gen)
        Ds = [int(x) for x in os.environ["KB_D"].split(",")] if os.environ.get("KB_D") else (6, 8, 32, 64, 128)
        for D in Ds:                                                 # D = 6: the flat word kernel k_gatherE
            rows, n = T // D, (1 << 30) // (4 * D)                     # 1 GiB of gathered rows
            devmem.view(b + 2 * GiB + GiB // 2, n, torch.int32).random_(0, rows, generator=gen)
            r = time_modes(lambda m, s: arena.gather(p.id, m, b + 3 * GiB, b, b + 2 * GiB + GiB // 2, n, D, stream=s),
                           args.reps)
            results[f"gather_rows_D{D}"] = summarize(f"gather rows D={D} ({4 * D} B)", r, 4 * n + 8 * n * D,
                                                     "GB/s", hbm)

    if want("stencil"):
        H = W = 32768
        devmem.view(b + 4 * GiB, H * W, torch.float32).uniform_(0, 1, generator=gen)
        r = time_modes(lambda m, s: arena.stencil(p.id, m, b + 8 * GiB, b + 4 * GiB, H, W, W, 0.5, 0.125, stream=s),
                       args.reps)
        results["stencil_32768^2"] = summarize("stencil 32768^2", r, 8 * (H - 2) * (W - 2), "GB/s", hbm)

    if want("stencil_tma"):
        H = W = 32768
        devmem.view(b + 4 * GiB, H * W, torch.float32).uniform_(0, 1, generator=gen)
        r = time_modes(lambda m, s: arena.stencil_tma(p.id, m, b + 8 * GiB, b + 4 * GiB, H, W, W, 0.5, 0.125,
                                                      stream=s), args.reps)
        results["stencil_tma_32768^2"] = summarize("stencil v2 (TMA) 32768^2", r, 8 * (H - 2) * (W - 2), "GB/s",
                                                   hbm)

    if only is not None and "l2" in only:
        # L2-resident working sets (< 126 MB L2), where the
        # fence's ALU cost is least hidden (the paper's all-cache-hit worst case,
        # 28-57 % at 100 % L1 hits)
        MiB = 1 << 20
        b = p.base + int(os.environ.get("KB_L2_OFF", "0"))   # placement probe (bench.py uses base + 1 GiB)
        devmem.view(b, 16 * MiB, torch.int32).random_(generator=gen)
        r = time_modes_batched(lambda m, s: arena.copy(p.id, m, b + 64 * MiB, b, 32 * MiB, stream=s), args.reps)
        results["l2_copy_32MiB"] = summarize("L2 copy 32 MiB", r, 2 * 32 * MiB, "GB/s", hbm)
        devmem.view(b + 128 * MiB, 8 * MiB, torch.float32).uniform_(-1, 1, generator=gen)
        devmem.view(b + 192 * MiB, 8 * MiB, torch.float32).uniform_(-1, 1, generator=gen)
        r = time_modes_batched(lambda m, s: arena.saxpy(p.id, m, 1.0, b + 128 * MiB, b + 192 * MiB, 8 * MiB,
                                                        stream=s), args.reps)
        results["l2_saxpy_8M"] = summarize("L2 saxpy 2^23", r, 12 * 8 * MiB, "GB/s", hbm)
        n, T = 1 << 22, 1 << 22                      # 16 MiB table, 16 MiB indices: L2-resident
        devmem.view(b + 256 * MiB, n, torch.int32).random_(0, T, generator=gen)
        r = time_modes_batched(lambda m, s: arena.gather(p.id, m, b + 320 * MiB, b, b + 256 * MiB, n, stream=s),
                               args.reps)
        results["l2_gather_4M"] = summarize("L2 gather 2^22 into 2^22", r, 12 * n, "GB/s", hbm)
        H = W = 2048                                 # 16 MiB in + out
        devmem.view(b + 384 * MiB, H * W, torch.float32).uniform_(0, 1, generator=gen)
        r = time_modes_batched(lambda m, s: arena.stencil(p.id, m, b + 448 * MiB, b + 384 * MiB, H, W, W, 0.5, 0.125,
                                                          stream=s), args.reps)
        results["l2_stencil_2048^2"] = summarize("L2 stencil 2048^2", r, 8 * (H - 2) * (W - 2), "GB/s", hbm)
        # K5 v2 at the same L2-resident size: the fence lives in the tensor maps
        r = time_modes_batched(lambda m, s: arena.stencil_tma(p.id, m, b + 448 * MiB, b + 384 * MiB, H, W, W, 0.5,
                                                              0.125, stream=s), args.reps)
        results["l2_stencil_tma_2048^2"] = summarize("L2 stencil v2 (TMA) 2048^2", r, 8 * (H - 2) * (W - 2), "GB/s",
                                                     hbm)

    if want("gemm"):
        n = 8192
        A, B, C = b, b + n * n * 2, b + 2 * n * n * 2
        devmem.view(A, n * n, torch.bfloat16).uniform_(-1, 1, generator=gen)
        devmem.view(B, n * n, torch.bfloat16).uniform_(-1, 1, generator=gen)
        ta = devmem.view(A, n * n, torch.bfloat16).view(n, n)
        tb = devmem.view(B, n * n, torch.bfloat16).view(n, n)
        tc = torch.empty(n, n, dtype=torch.bfloat16, device="cuda")
        r = time_modes(lambda m, s: arena.gemm(p.id, m, C, A, B, n, n, n, n, n, n, stream=s), args.reps,
                       extra={"torch": lambda s: torch.matmul(ta, tb.t(), out=tc)})
        xs = r.pop("torch")
        res = summarize("gemm 8192^3 bf16", r, 2 * n ** 3, "TFLOP/s", bf16)
        res["torch_matmul"] = {"ms_median": round(statistics.median(xs), 4),
                               "TFLOP/s": round(2 * n ** 3 / (statistics.median(xs) / 1e3) / 1e12, 1),
                               "note": "cuBLAS via torch.matmul, timed interleaved with the fenced GEMM"}
        print(f"  torch.matmul: {res['torch_matmul']['TFLOP/s']} TFLOP/s", file=sys.stderr)
        results["gemm_8192^3"] = res
    results["device_flags"] = arena.device_flags()
    print(json.dumps(results))
    arena.close()


if __name__ == "__main__":
    main()
