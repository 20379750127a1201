"""Launch one fenced kernel a few times on a single tenant partition (for ncu).

  python tools/prof_kernel.py --kind saxpy --mode mask [--reps 3]
  python tools/prof_kernel.py --kind gatherrows --D 32 --mode check
Sizes are the bench's per-tenant sizes (4 GiB tensors; C3 gather; 8192^3 GEMM;
32768^2 stencil; kernel_bench's 1 GiB of gathered D-word rows) in a 16 GiB
partition.
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2401_09290_b200 import devmem, guardian as g  # noqa: E402

GiB = 1 << 30


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--kind", default="saxpy")
    ap.add_argument("--mode", default="mask")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--D", type=int, default=32, help="row width (words) for --kind gatherrows")
    ap.add_argument("--pa", action="store_true", help="per-access fencing (GD_FENCE_PER_ACCESS)")
    ap.add_argument("--l2", action="store_true", help="stencil at the L2-resident size 2048^2")
    ap.add_argument("--oob", type=float, default=0.01, help="gather / scatter: fraction of planted out-of-partition indices")
    a = ap.parse_args()
    if a.pa:
        a.mode += "+pa"
    ar = g.Arena(0, 1 << 34)
    p = ar.partition_alloc(1 << 34)
    gen = torch.Generator(device="cuda:0")
    gen.manual_seed(2000)
    b = p.base
    if a.kind in ("gather", "scatter"):
        # C3: uniform in-bounds indices into the 2^29-entry table, 1 % planted below the base
        idx = devmem.view(b + 2 * GiB, 1 << 26, torch.int32)
        idx.random_(0, 1 << 29, generator=gen)
        pos = torch.randperm(1 << 26, generator=gen, device="cuda:0")[: int((1 << 26) * a.oob)]
        idx[pos] = torch.randint(-2**31, 0, (pos.numel(),), generator=gen, device="cuda:0", dtype=torch.int32)
        devmem.view(b, 1 << 29, torch.int32).random_(generator=gen)
    if a.kind == "gatherrows":
        T = 1 << 29
        rows, n_rows = T // a.D, GiB // (4 * a.D)
        devmem.view(b, T, torch.int32).random_(generator=gen)
        devmem.view(b + 2 * GiB + GiB // 2, n_rows, torch.int32).random_(0, rows, generator=gen)
    for _ in range(a.reps):
        if a.kind == "copy":
            ar.copy(p.id, a.mode, b + 4 * GiB, b, 4 * GiB)
        elif a.kind == "saxpy":
            ar.saxpy(p.id, a.mode, 1.5, b + 8 * GiB, b + 12 * GiB, 1 << 30)
        elif a.kind == "gather":
            ar.gather(p.id, a.mode, b + 2 * GiB + GiB // 4, b, b + 2 * GiB, 1 << 26)
        elif a.kind == "gatherrows":
            ar.gather(p.id, a.mode, b + 3 * GiB, b, b + 2 * GiB + GiB // 2, n_rows, a.D)
        elif a.kind == "scatter":
            ar.scatter(p.id, a.mode, b, b + 2 * GiB, b + 2 * GiB + GiB // 4, 1 << 26)
        elif a.kind == "stencil_tma":
            ar.stencil_tma(p.id, a.mode, b + 8 * GiB, b + 4 * GiB, 32768, 32768, 32768, 0.5, 0.125)
        elif a.kind == "stencil":
            hw = 2048 if a.l2 else 32768
            ar.stencil(p.id, a.mode, b + 8 * GiB, b + 4 * GiB, hw, hw, hw, 0.5, 0.125)
        elif a.kind == "gemm":
            n = 8192
            ar.gemm(p.id, a.mode, b + 2 * n * n * 2, b, b + n * n * 2, n, n, n, n, n, n)
    torch.cuda.synchronize()
    print("flags", ar.device_flags())
    ar.close()


if __name__ == "__main__":
    main()
