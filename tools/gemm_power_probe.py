"""Clock / power under the cap: back-to-back 8192^3 bf16 GEMMs for a few
seconds, ours (fenced, mask) vs cuBLAS (torch.matmul), sampling nvidia-smi
(dev probe; the power-cap explanation of the GEMM gap in DESIGN.md)."""
import os
import subprocess
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2401_09290_b200 import devmem, guardian as g  # noqa: E402


def sample(fn, secs=4.0):
    q = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,power.draw,temperature.gpu",
                          "--format=csv,noheader,nounits", "-lms", "100"], stdout=subprocess.PIPE, text=True)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 0
    t0 = time.time()
    s.record()
    while time.time() - t0 < secs:
        for _ in range(20):
            fn()
        n += 20
        torch.cuda.synchronize()
    e.record()
    e.synchronize()
    q.terminate()
    rows = [r.split(",") for r in q.stdout.read().strip().splitlines()]
    rows = rows[len(rows) // 3:]                                   # steady state
    clk = sorted(float(r[0]) for r in rows)
    pw = sorted(float(r[1]) for r in rows)
    ms = s.elapsed_time(e) / n
    return {"ms": round(ms, 4), "TFLOP/s": round(2 * 8192 ** 3 / ms / 1e9, 1), "sm_mhz_median": clk[len(clk) // 2],
            "power_w_median": pw[len(pw) // 2], "samples": len(rows)}


def main():
    n = 8192
    a = g.Arena(0, 1 << 34)
    p = a.partition_alloc(1 << 34)
    gen = torch.Generator(device="cuda")
    gen.manual_seed(1)
    for off in (0, n * n * 2):
        devmem.view(p.base + off, n * n, torch.bfloat16).uniform_(-1, 1, generator=gen)
    A = torch.randn(n, n, dtype=torch.bfloat16, device="cuda")
    B = torch.randn(n, n, dtype=torch.bfloat16, device="cuda")
    ours = lambda: a.gemm(p.id, "mask", p.base + 2 * n * n * 2, p.base, p.base + n * n * 2, n, n, n, n, n, n)
    cublas = lambda: torch.matmul(A, B.t())
    for _ in range(2):
        for name, fn in (("ours", ours), ("cublas", cublas)):
            print(name, sample(fn), flush=True)


if __name__ == "__main__":
    main()
