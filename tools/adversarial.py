"""Adversarial tenant: gathers (single words and 128-bit rows), scatter-adds,
copies, SAXPYs, stencils and GEMMs through arbitrary int32 indices and raw
pointers into other tenants' memory and far outside the arena.  Run under compute-sanitizer by tests/test_gpu_isolation.py:
fenced modes must produce no invalid access at all; the unfenced twin
(--mode none) must be flagged (it would corrupt or fault the shared context,
which is why it only ever runs in a subprocess).

  python tools/adversarial.py --mode mask|modulo|check|maskcount|clamp|none
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2401_09290_b200 import devmem, guardian as g  # noqa: E402

MiB = 1 << 20


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--mode", default="mask")
    args = ap.parse_args()
    a = g.Arena(0, 4 * 16 * MiB)
    parts = [a.partition_alloc(16 * MiB) for _ in range(4)]
    p = parts[1]
    rng = synth.rng_for(777)
    n = 1 << 16
    j = synth.chaos_indices(rng, n)
    devmem.view(p.base + 4 * MiB, n, torch.int32).copy_(torch.from_numpy(j))
    a.gather(p.id, args.mode, p.base + 6 * MiB, p.base, p.base + 4 * MiB, n)
    a.scatter(p.id, args.mode, p.base, p.base + 4 * MiB, p.base + 6 * MiB, n)
    a.gather(p.id, args.mode, p.base + 6 * MiB, p.base, p.base + 4 * MiB, n // 32, 32)      # 128-B rows
    far = int(rng.integers(1 << 40, 1 << 47)) & ~15
    for src in (parts[0].base + 4096, 0x10, far):
        a.copy(p.id, args.mode, p.base + 8 * MiB, src, 64 * 1024)
        a.saxpy(p.id, args.mode, 0.5, src, p.base + 8 * MiB, 16 * 1024)                  # x elsewhere
        a.saxpy(p.id, args.mode, 0.5, p.base + 8 * MiB, src, 16 * 1024)                  # y elsewhere
        a.stencil(p.id, args.mode, src, p.base + 8 * MiB, 40, 200, 200, 0.5, 0.125)       # out elsewhere
        a.stencil(p.id, args.mode, p.base + 8 * MiB, src, 40, 200, 200, 0.5, 0.125)       # in elsewhere
        if args.mode != "none":                    # unfenced TMA would fault the context outright
            a.stencil_tma(p.id, args.mode, src, p.base + 8 * MiB, 40, 203, 204, 0.5, 0.125)
            a.stencil_tma(p.id, args.mode, p.base + 8 * MiB, src, 40, 203, 204, 0.5, 0.125)
    if args.mode != "none":                        # the unfenced GEMM's TMA would fault the context outright
        for src in (parts[0].base + 4096, far):
            a.gemm(p.id, args.mode, p.base + 10 * MiB, src, p.base + 12 * MiB, 256, 256, 128, 128, 128, 256)
            a.gemm(p.id, args.mode, src, p.base + 12 * MiB, p.base + 12 * MiB, 256, 256, 128, 128, 128, 256)
    torch.cuda.synchronize()
    print("done", args.mode, a.stats(p.id)["violations"])


if __name__ == "__main__":
    main()
