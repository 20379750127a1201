"""Placement / process-state probe of the L2-resident per-access D = 1 gather
(DESIGN.md §12): the same 2^22-index gather into a 16 MiB table on tenant 7
of an 8 x 16 GiB arena, either inside bench.py's Workload (8 partitions of
C2 data written) or in a plain arena.

  python tools/l2_gather_probe.py bench_ws|plain [mode ...]   # time the modes
  python tools/l2_gather_probe.py bench_ws|plain --once MODE  # 3 launches (ncu)
"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import torch  # noqa: E402

import bench  # noqa: E402
import kernel_bench as kb  # noqa: E402
from paper_2401_09290_b200 import devmem  # noqa: E402

MiB = 1 << 20


def main():
    torch.cuda.set_device(0)
    kind = sys.argv[1]
    if kind == "bench_ws":
        w = bench.Workload(0)
        a, p = w.arena, w.parts[7]
    else:
        from paper_2401_09290_b200 import guardian as g
        a = g.Arena(0, 1 << 37)
        parts = [a.partition_alloc(1 << 34) for _ in range(8)]
        p = parts[7]
    b = p.base + (1 << 30)
    gen = torch.Generator(device="cuda:0")
    gen.manual_seed(5207)
    devmem.view(b, 8 * MiB, torch.int32).random_(generator=gen)
    n = 1 << 22
    devmem.view(b + 256 * MiB, n, torch.int32).random_(0, n, generator=gen)
    torch.cuda.synchronize()
    launch = lambda m, s=None: a.gather(p.id, m, b + 320 * MiB, b, b + 256 * MiB, n, stream=s)  # noqa: E731
    if "--once" in sys.argv:
        m = sys.argv[sys.argv.index("--once") + 1]
        for _ in range(3):
            launch(m)
        torch.cuda.synchronize()
        return
    kb.MODES[:] = sys.argv[2:] or ["none", "mask", "check", "check+pa", "modulo+pa"]
    r = kb.time_modes_batched(launch, 12)
    base = statistics.median(r["none"])
    print(kind, {m: round(100 * (statistics.median(v) / base - 1), 2) for m, v in r.items()})


if __name__ == "__main__":
    main()
