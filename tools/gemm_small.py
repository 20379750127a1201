"""One small fenced GEMM on each path (2-SM for >= 256 rows, 1-SM below) and
both stencils, for compute-sanitizer racecheck / synccheck runs (dev tool):
  compute-sanitizer --tool racecheck python tools/gemm_small.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2401_09290_b200 import devmem, guardian as g  # noqa: E402

MiB = 1 << 20


def main():
    a = g.Arena(0, 32 * MiB)
    p = a.partition_alloc(16 * MiB)
    gen = torch.Generator(device="cuda")
    gen.manual_seed(3)
    devmem.view(p.base, 4 * MiB, torch.bfloat16).uniform_(-1, 1, generator=gen)
    for M in (512, 128):
        a.gemm(p.id, "mask", p.base + 8 * MiB, p.base, p.base + 2 * MiB, M, 256, 256, 256, 256, 256)
    devmem.view(p.base + 4 * MiB, 1 << 20, torch.float32).uniform_(0, 1, generator=gen)
    a.stencil(p.id, "check", p.base + 12 * MiB, p.base + 4 * MiB, 200, 1000, 1024, 0.5, 0.125)
    a.stencil_tma(p.id, "check", p.base + 12 * MiB, p.base + 4 * MiB, 200, 1001, 1024, 0.5, 0.125)
    torch.cuda.synchronize()
    print("flags", a.device_flags())


if __name__ == "__main__":
    main()
