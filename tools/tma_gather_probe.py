"""Time tools/tma_gather_probe.cu (TMA tile::gather4 per L2 promotion vs an
LSU load gather) on the C3 shape and check the results agree (dev probe).
Run the DRAM-bytes side under ncu:
  ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum -k regex:k_ python tools/tma_gather_probe.py --once
"""
import ctypes
import os
import statistics
import subprocess
import sys

import torch

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "libtmagather.so")


def main():
    if not os.path.exists(LIB):
        subprocess.check_call(["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3",
                               "-shared", "-Xcompiler", "-fPIC", "-o", LIB, os.path.join(HERE, "tma_gather_probe.cu"),
                               "-L/usr/local/cuda/lib64/stubs", "-lcuda"])
    L = ctypes.CDLL(LIB)
    L.tg_run.argtypes = [ctypes.c_int] + [ctypes.c_uint64] * 5 + [ctypes.c_void_p]
    L.ld_run.argtypes = [ctypes.c_uint64] * 4 + [ctypes.c_void_p]
    once = "--once" in sys.argv
    n, T = 1 << 26, 1 << 29
    g = torch.Generator(device="cuda")
    g.manual_seed(7)
    table = torch.randint(-2**31, 2**31 - 1, (T,), dtype=torch.int32, device="cuda", generator=g)
    idx = torch.randint(0, T, (n,), dtype=torch.int32, device="cuda", generator=g)
    out_ref = torch.empty(n, dtype=torch.int32, device="cuda")
    out = torch.empty(n, dtype=torch.int32, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    assert L.ld_run(table.data_ptr(), idx.data_ptr(), out_ref.data_ptr(), n, s) == 0
    torch.cuda.synchronize()
    assert torch.equal(out_ref, table[idx.long()])
    runs = [("lsu ldcg", lambda: L.ld_run(table.data_ptr(), idx.data_ptr(), out.data_ptr(), n, s))]
    for p, name in enumerate(("none", "64B", "128B", "256B")):
        runs.append((f"tma gather4 promo {name}",
                     lambda p=p: L.tg_run(p, table.data_ptr(), T // 4, idx.data_ptr(), out.data_ptr(), n, s)))
    for name, fn in runs:
        out.zero_()
        rc = fn()
        torch.cuda.synchronize()
        assert rc == 0, (name, rc)
        assert torch.equal(out, out_ref), name
        if once:
            continue
        ts = []
        for i in range(13):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            fn()
            b.record()
            b.synchronize()
            if i >= 3:
                ts.append(a.elapsed_time(b))
        ms = statistics.median(ts)
        print(f"{name:24s} {ms:8.4f} ms  {n / ms / 1e6:7.2f} Gidx/s  {12 * n / ms / 1e6:8.1f} GB/s alg", flush=True)


if __name__ == "__main__":
    main()
