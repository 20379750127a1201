"""C5 (BASELINE configs[4]) makespan under different issue policies (dev probe):
8 tenant streams round-robin (the launcher's default), one stream (time-
sharing), and GEMM grids capped at fewer SMs (GD_GEMM_MAX_SMS, set per run by
the caller).  Prints makespan and the serial sum of solo kernel times.
  python tools/c5_policies.py [--launches 20]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import bench  # noqa: E402


def makespan(w, queue, streams, policy="round_robin"):
    torch = w.torch
    root = torch.cuda.current_stream(w.device)
    start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(w.device)
    start.record(root)
    for s in streams:
        s.wait_event(start)
    w.arena.launcher_run(queue, streams, policy=policy)
    for s in streams:
        e = torch.cuda.Event()
        e.record(s)
        root.wait_event(e)
    stop.record(root)
    torch.cuda.synchronize(w.device)
    return start.elapsed_time(stop)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--launches", type=int, default=20)
    a = ap.parse_args()
    w = bench.Workload(0)
    ms, nbytes, flops, planted = w.c5(launches=a.launches)          # builds the C5 inputs; the bench's own number
    print(f"bench c5 (8 streams, round robin): {ms:.1f} ms", flush=True)
    # rebuild the item list exactly as c5 does (its inputs are in place now)
    g = w.g
    items = []
    n_idx, n = 1 << 26, 8192
    for t, p in enumerate(w.parts):
        b = p.base
        if t < 3:
            items.append(g.work(p.id, g.GD_KIND_COPY, "check", ptr=(b + bench.OFF_DST, b + bench.OFF_SRC),
                                u64=(bench.COPY_BYTES,)))
        elif t < 6:
            items.append(g.work(p.id, g.GD_KIND_GATHER, "check", ptr=(b + 2 * bench.GiB + bench.GiB // 4, b,
                                                                      b + 2 * bench.GiB), u64=(n_idx,), u32=(1,)))
        else:
            items.append(g.work(p.id, g.GD_KIND_GEMM, "check", ptr=(b + 2 * n * n * 2, b, b + n * n * 2),
                                u64=(n, n, n), u32=(n, n, n)))
    queue = [it for it in items for _ in range(a.launches)]
    solo = {}
    for name, it in (("copy", items[0]), ("gather", items[3]), ("gemm", items[6])):
        for _ in range(2):
            makespan(w, [it] * 5, w.streams[:1])
        solo[name] = makespan(w, [it] * 10, w.streams[:1]) / 10
    serial_sum = a.launches * (3 * solo["copy"] + 3 * solo["gather"] + 2 * solo["gemm"])
    print(f"solo ms: {solo}; serial sum {serial_sum:.1f} ms", flush=True)
    for label, streams, pol in (("8 streams", w.streams, "round_robin"), ("1 stream", w.streams[:1], "round_robin"),
                                ("8 streams no_tensor_random", w.streams, "no_tensor_random"),
                                ("8 streams memory_lane", w.streams, "memory_lane")):
        makespan(w, queue[:16], streams, pol)
        ts = sorted(makespan(w, queue, streams, pol) for _ in range(3))
        print(f"{label:28s} makespan {ts[1]:7.1f} ms  (serial sum {serial_sum:.1f})", flush=True)
    # pairwise interference: two tenants of two kinds, concurrent (2 streams) vs serial (1 stream)
    kinds = {"copy": items[0], "gather": items[3], "gemm": items[6]}
    for x, y in (("copy", "gather"), ("copy", "gemm"), ("gather", "gemm"), ("copy", "copy"), ("gather", "gather")):
        ix, iy = kinds[x], kinds[y]
        if x == y:
            iy = items[1] if x == "copy" else items[4]
        q = [ix] * 10 + [iy] * 10
        conc = sorted(makespan(w, q, w.streams[:2]) for _ in range(3))[1]
        ser = sorted(makespan(w, q, w.streams[:1]) for _ in range(3))[1]
        print(f"pair {x:6s}+{y:6s}: concurrent {conc:6.1f} ms  serial {ser:6.1f} ms  ({100 * (conc / ser - 1):+.1f} %)",
              flush=True)


if __name__ == "__main__":
    main()
