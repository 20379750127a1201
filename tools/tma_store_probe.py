"""Which TMA store boxes are legal (dev probe): each case in a fresh process."""
import ctypes, os, subprocess, sys
HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "libtmastore.so")
CASES = [(32, 32, 0, 1, 1), (32, 32, 1, 1, 1), (64, 32, 1, 1, 1), (128, 32, 1, 1, 1), (252, 32, 1, 1, 1),
         (256, 32, 1, 1, 1), (252, 32, 1, 0, 0), (32, 32, 1, 0, 0), (8, 8, 1, 1, 1), (252, 8, 1, 1, 1)]
if len(sys.argv) > 1:
    import torch
    L = ctypes.CDLL(LIB)
    L.st_run.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint32,
                         ctypes.c_uint32, ctypes.c_int, ctypes.c_int, ctypes.c_int]
    bw, bh, f32, x0, y0 = map(int, sys.argv[1:6])
    buf = torch.zeros(1 << 22, dtype=torch.float32, device="cuda")
    print(L.st_run(buf.data_ptr(), 1000, 1000, 1024, bw, bh, f32, x0, y0))
else:
    if not os.path.exists(LIB):
        subprocess.check_call(["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-shared",
                               "-Xcompiler", "-fPIC", "-o", LIB, os.path.join(HERE, "tma_store_probe.cu"),
                               "-L/usr/local/cuda/lib64/stubs", "-lcuda"])
    for c in CASES:
        r = subprocess.run([sys.executable, __file__] + [str(x) for x in c], capture_output=True, text=True)
        print(c, (r.stdout.strip() or r.stderr.strip()[-120:]))
