"""Adversarial tenant: gathers, scatter-adds and copies through arbitrary
int32 indices and raw pointers into other tenants' memory and far outside
the arena.  Run under compute-sanitizer by tests/test_gpu_isolation.py:
fenced modes must produce no invalid access at all; the unfenced twin
(--mode none) must be flagged (it would corrupt or fault the shared context,
which is why it only ever runs in a subprocess).

  python tools/adversarial.py --mode mask|modulo|check|none
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
    for src in (parts[0].base + 4096, 0x10, int(rng.integers(1 << 40, 1 << 47)) & ~15):
        a.copy(p.id, args.mode, p.base + 8 * MiB, src, 64 * 1024)
    torch.cuda.synchronize()
    print("done", args.mode, a.stats(p.id)["violations"])


if __name__ == "__main__":
    main()
