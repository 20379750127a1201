import os, sys, json
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tools')
import bench, torch
import kernel_bench as kb
from paper_2401_09290_b200 import devmem
torch.cuda.set_device(0)
MiB = 1 << 20
mode = sys.argv[1]
if mode == "bench_ws":
    w = bench.Workload(0)
    a, p = w.arena, w.parts[7]
else:
    from paper_2401_09290_b200 import guardian as g
    a = g.Arena(0, 1 << 37); parts = [a.partition_alloc(1 << 34) for _ in range(8)]; p = parts[7]
b = p.base + (1 << 30)
gen = torch.Generator(device="cuda:0"); gen.manual_seed(5207)
devmem.view(b, 8 * MiB, torch.int32).random_(generator=gen)
n = 1 << 22
devmem.view(b + 256 * MiB, n, torch.int32).random_(0, n, generator=gen)
torch.cuda.synchronize()
kb.MODES[:] = ["none", "mask", "check", "check+pa", "modulo+pa"]
r = kb.time_modes_batched(lambda m, s: a.gather(p.id, m, b + 320 * MiB, b, b + 256 * MiB, n, stream=s), 12)
import statistics
base = statistics.median(r["none"])
print(mode, {m: round(100 * (statistics.median(v) / base - 1), 2) for m, v in r.items()})
