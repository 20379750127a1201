"""Host<->device transfer ceiling on the box (for bench.py's e2e leg):
torch copies and the checked gd_memcpy_h2d / d2h from pinned host memory,
one direction at a time and both directions concurrently.

  python tools/pcie_probe.py
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2401_09290_b200 import guardian as g  # noqa: E402

GiB = 1 << 30
N = 4 * GiB


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps


def main():
    hin = torch.empty(N, dtype=torch.uint8, pin_memory=True)
    hout = torch.empty(N, dtype=torch.uint8, pin_memory=True)
    hin.random_(0, 256)
    dev = torch.empty(N, dtype=torch.uint8, device="cuda")
    dev2 = torch.empty(N, dtype=torch.uint8, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    res = {}
    res["torch_h2d"] = N / timed(lambda: dev.copy_(hin, non_blocking=True)) / 1e9
    res["torch_d2h"] = N / timed(lambda: hout.copy_(dev, non_blocking=True)) / 1e9

    def both():
        with torch.cuda.stream(s1):
            dev.copy_(hin, non_blocking=True)
        with torch.cuda.stream(s2):
            hout.copy_(dev2, non_blocking=True)
    res["torch_both_GBps_total"] = 2 * N / timed(both) / 1e9
    a = g.Arena(0, 1 << 34)
    p = a.partition_alloc(1 << 34)
    res["gd_h2d"] = N / timed(lambda: a.memcpy_h2d(p.id, p.base, hin.data_ptr(), N, stream=s1)) / 1e9
    res["gd_d2h"] = N / timed(lambda: a.memcpy_d2h(p.id, hout.data_ptr(), p.base, N, stream=s1)) / 1e9

    def gboth():
        a.memcpy_h2d(p.id, p.base, hin.data_ptr(), N, stream=s1)
        a.memcpy_d2h(p.id, hout.data_ptr(), p.base + N, N, stream=s2)
    res["gd_both_GBps_total"] = 2 * N / timed(gboth) / 1e9
    # many smaller concurrent uploads on 8 streams (the e2e leg's pattern)
    ss = [torch.cuda.Stream() for _ in range(8)]

    def multi():
        for i, s in enumerate(ss):
            a.memcpy_h2d(p.id, p.base + i * (N // 8), hin.data_ptr() + i * (N // 8), N // 8, stream=s)
    res["gd_h2d_8streams"] = N / timed(multi) / 1e9
    for k, v in res.items():
        print(f"{k:24s} {v:8.2f} GB/s")


if __name__ == "__main__":
    main()
