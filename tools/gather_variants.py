"""Time gather_variants.cu on the C3 shape (2^26 random indices into 2^29 u32),
plus an ncu-free DRAM estimate from the timing (dev probe)."""
import ctypes
import json
import os
import statistics
import subprocess
import sys

import torch

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "libgvariants.so")


def main():
    if not os.path.exists(LIB):
        subprocess.check_call(["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3",
                               "-shared", "-Xcompiler", "-fPIC", "-o", LIB, os.path.join(HERE, "gather_variants.cu")])
    L = ctypes.CDLL(LIB)
    L.gvariant_name.restype = ctypes.c_char_p
    L.gvariant_run.argtypes = [ctypes.c_int] + [ctypes.c_uint64] * 6 + [ctypes.c_void_p]
    P = 1 << 34
    buf = torch.empty(2 * P, dtype=torch.uint8, device="cuda")
    base = (buf.data_ptr() + P - 1) & ~(P - 1)
    n, T = 1 << 26, 1 << 29
    table, idx, out = base, base + (2 << 30), base + (2 << 30) + (1 << 28)
    tv = torch.as_tensor(buf[table - buf.data_ptr():table - buf.data_ptr() + 4 * T]).view(torch.int32)
    tv.random_()
    iv = torch.as_tensor(buf[idx - buf.data_ptr():idx - buf.data_ptr() + 4 * n]).view(torch.int32)
    iv.random_(0, T)
    s = torch.cuda.current_stream()
    res = {}
    L.svariant_run.argtypes = [ctypes.c_uint64] * 6 + [ctypes.c_void_p]
    src = out + (1 << 28)
    print("default L2 fetch granularity", L.get_l2_fetch(), file=sys.stderr)
    for gran in (0, 32, 64, 128):
        if gran:
            L.set_l2_fetch(gran)
        got = L.get_l2_fetch()
        for name, fn in (("gather ldcg U2", lambda: L.gvariant_run(1, base, P - 1, out, table, idx, n, s.cuda_stream)),
                         ("scatter U4", lambda: L.svariant_run(base, P - 1, table, idx, src, n, s.cuda_stream))):
            ts = []
            for i in range(13):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                assert fn() == 0
                b.record()
                b.synchronize()
                if i >= 3:
                    ts.append(a.elapsed_time(b))
            ms = statistics.median(ts)
            key = f"{name} l2fetch={got}"
            res[key] = {"ms": round(ms, 4), "Gidx_per_s": round(n / (ms / 1e3) / 1e9, 2)}
            print(f"{key:34s} {ms:8.4f} ms {res[key]['Gidx_per_s']} Gidx/s", file=sys.stderr)
    L.set_l2_fetch(128)
    L.rread_run.argtypes = [ctypes.c_int, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_void_p,
                            ctypes.c_void_p]
    sink = torch.zeros(4, dtype=torch.int32, device="cuda")
    iv.random_()
    for wb in (4, 8, 16, 32, 64, 128):
        ts = []
        for i in range(13):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            assert L.rread_run(wb, table, idx, n, sink.data_ptr(), s.cuda_stream) == 0
            b.record()
            b.synchronize()
            if i >= 3:
                ts.append(a.elapsed_time(b))
        ms = statistics.median(ts)
        key = f"random read {wb} B"
        res[key] = {"ms": round(ms, 4), "Gaccess_per_s": round(n / (ms / 1e3) / 1e9, 2),
                    "useful_GBps": round(n * wb / (ms / 1e3) / 1e9, 1)}
        print(f"{key:24s} {ms:8.4f} ms {res[key]['Gaccess_per_s']} Gacc/s {res[key]['useful_GBps']} GB/s useful",
              file=sys.stderr)
    for v in range(L.gvariant_count()):
        ts = []
        for i in range(13):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            rc = L.gvariant_run(v, base, P - 1, out, table, idx, n, s.cuda_stream)
            b.record()
            b.synchronize()
            assert rc == 0, rc
            if i >= 3:
                ts.append(a.elapsed_time(b))
        ms = statistics.median(ts)
        name = L.gvariant_name(v).decode()
        res[name] = {"ms": round(ms, 4), "alg_GBps": round(12 * n / (ms / 1e3) / 1e9, 1),
                     "Gidx_per_s": round(n / (ms / 1e3) / 1e9, 2)}
        print(f"{name:20s} {ms:8.4f} ms {res[name]['alg_GBps']:8.1f} GB/s alg  {res[name]['Gidx_per_s']} Gidx/s",
              file=sys.stderr)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
