"""Time the stream_variants.cu copy variants on a 4 GiB copy (dev probe).

  python tools/stream_variants.py   (builds tools/libvariants.so if needed)
"""
import ctypes
import os
import statistics
import subprocess
import sys

import torch

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "libvariants.so")


def main():
    if not os.path.exists(LIB):
        subprocess.check_call(["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3",
                               "-shared", "-Xcompiler", "-fPIC", "-o", LIB, os.path.join(HERE, "stream_variants.cu")])
    L = ctypes.CDLL(LIB)
    L.variant_name.restype = ctypes.c_char_p
    L.variant_copy.argtypes = [ctypes.c_int] + [ctypes.c_uint64] * 5 + [ctypes.c_void_p]
    n = 4 << 30
    buf = torch.empty(2 * n + (1 << 34), dtype=torch.uint8, device="cuda")   # room to align a 16 GiB "partition"
    base = (buf.data_ptr() + (1 << 34) - 1) & ~((1 << 34) - 1)
    if base + 2 * n > buf.data_ptr() + buf.numel():
        base = buf.data_ptr()
    mask = (1 << 40) - 1 if base == buf.data_ptr() else (1 << 34) - 1
    src, dst = base, base + n
    s = torch.cuda.current_stream()
    res = {}
    for v in range(L.variant_count()):
        ts = []
        for i in range(13):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            rc = L.variant_copy(v, base & ~mask, mask, dst, src, n, s.cuda_stream)
            b.record()
            b.synchronize()
            assert rc == 0, rc
            if i >= 3:
                ts.append(a.elapsed_time(b))
        ms = statistics.median(ts)
        res[L.variant_name(v).decode()] = round(2 * n / (ms / 1e3) / 1e9, 1)
        print(f"{L.variant_name(v).decode():24s} {res[L.variant_name(v).decode()]:8.1f} GB/s", file=sys.stderr)
    # torch reference
    x = torch.empty(n, dtype=torch.uint8, device="cuda")
    y = torch.empty_like(x)
    ts = []
    for i in range(13):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        y.copy_(x)
        b.record()
        b.synchronize()
        if i >= 3:
            ts.append(a.elapsed_time(b))
    res["torch copy_"] = round(2 * n / (statistics.median(ts) / 1e3) / 1e9, 1)
    print(f"{'torch copy_':24s} {res['torch copy_']:8.1f} GB/s", file=sys.stderr)
    import json
    print(json.dumps(res))


if __name__ == "__main__":
    main()
