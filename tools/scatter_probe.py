"""Time tools/scatter_probe.cu (dev probe): random read / store / RED / RMW
flavours over 2^26 uniform indices, table sizes from DRAM-resident (2 GiB)
to L2-resident (8 MiB).  Prints one JSON object; a text table on stderr.

  python tools/scatter_probe.py > gpurun_out/scatter_probe.json
"""
import ctypes
import json
import os
import statistics
import subprocess
import sys

import torch

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "libscatter_probe.so")


def main():
    src_cu = os.path.join(HERE, "scatter_probe.cu")
    if not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(src_cu):
        subprocess.check_call(["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3",
                               "-shared", "-Xcompiler", "-fPIC", "-o", LIB, src_cu])
    L = ctypes.CDLL(LIB)
    L.probe_name.restype = ctypes.c_char_p
    L.probe_run.argtypes = [ctypes.c_int, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64,
                            ctypes.c_uint32, ctypes.c_uint64, ctypes.c_void_p]
    n = 1 << 26
    table = torch.zeros(1 << 29, dtype=torch.int32, device="cuda")
    idx = torch.empty(n, dtype=torch.int32, device="cuda").random_()
    src = torch.empty(n, dtype=torch.int32, device="cuda").random_()
    sink = torch.zeros(4, dtype=torch.int32, device="cuda")
    s = torch.cuda.current_stream()
    res = {}
    for words_log in (29, 25, 24, 23, 21):
        words = 1 << words_log
        for k in range(L.probe_count()):
            name = L.probe_name(k).decode()
            ts = []
            for i in range(13):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                rc = L.probe_run(k, table.data_ptr(), idx.data_ptr(), src.data_ptr(), n, words, sink.data_ptr(),
                                 s.cuda_stream)
                b.record()
                b.synchronize()
                assert rc == 0, rc
                if i >= 3:
                    ts.append(a.elapsed_time(b))
            ms = statistics.median(ts)
            key = f"{name} table={4 * words >> 20}MiB"
            res[key] = {"ms": round(ms, 4), "Gidx_per_s": round(n / (ms / 1e3) / 1e9, 2),
                        "alg_GBps_16B": round(16 * n / (ms / 1e3) / 1e9, 1)}
            print(f"{key:34s} {ms:8.4f} ms {res[key]['Gidx_per_s']:7.2f} G/s  {res[key]['alg_GBps_16B']:8.1f} GB/s "
                  f"(16 B/idx)", file=sys.stderr)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
