"""CPU oracle for Guardian's per-access address fencing (arXiv 2401.09290).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
package.  The product path (``paper_2401_09290_b200``) never imports it, and
this package never imports the product: the two share no code.

The arithmetic lives in ``oracle.c`` (plain C11, ``-ffp-contract=off``); this
module only marshals arguments through ctypes, exactly like the product's
binding does for ``libguardian.so``.  ``alloc_ref.py`` holds the naive bitmap
partition allocator used to check the product allocator's invariants
("property test vs a naive bitmap allocator oracle").
"""
from __future__ import annotations

import ctypes
import threading
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "liboracle.so")

NONE, MASK, CHECK, MODULO, MASK_COUNT, CLAMP = 0, 1, 2, 3, 4, 5
MODES = {"none": NONE, "mask": MASK, "check": CHECK, "modulo": MODULO, "maskcount": MASK_COUNT, "clamp": CLAMP}


class OrCtx(ctypes.Structure):
    _fields_ = [
        ("va", ctypes.c_uint64),
        ("len", ctypes.c_uint64),
        ("bytes", ctypes.c_void_p),
        ("base", ctypes.c_uint64),
        ("size", ctypes.c_uint64),
        ("mode", ctypes.c_int32),
        ("pad_", ctypes.c_int32),
        ("violations", ctypes.c_uint64),
        ("faults", ctypes.c_uint64),
        ("accesses", ctypes.c_uint64),
    ]


_lib = None


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (plain C11, no fp contraction)."""
    src = os.path.join(_HERE, "oracle.c")
    hdr = os.path.join(_HERE, "oracle.h")
    if (not force and os.path.exists(LIB_PATH)
            and os.path.getmtime(LIB_PATH) >= max(os.path.getmtime(src), os.path.getmtime(hdr))):
        return LIB_PATH
    import subprocess
    tmp = f"{LIB_PATH}.{os.getpid()}.tmp"           # unique: concurrent builders never collide
    subprocess.check_call(["gcc", "-std=c11", "-O2", "-ffp-contract=off", "-fno-fast-math",
                           "-fPIC", "-shared", "-Wall", "-Wextra", "-o", tmp, src, "-lm"])
    os.replace(tmp, LIB_PATH)
    return LIB_PATH


_lib_lock = threading.Lock()


def lib():
    global _lib
    if _lib is not None:
        return _lib
    with _lib_lock:                      # threads of one process: build and load once
        if _lib is not None:
            return _lib
        build()
        L = ctypes.CDLL(LIB_PATH)
        u64, u32, f32, i32 = ctypes.c_uint64, ctypes.c_uint32, ctypes.c_float, ctypes.c_int
        P = ctypes.POINTER(OrCtx)
        L.or_mask.restype = u64
        L.or_mask.argtypes = [u64]
        L.or_fence_mask.restype = u64
        L.or_fence_mask.argtypes = [u64, u64, u64, u32]
        L.or_fence_modulo.restype = u64
        L.or_fence_modulo.argtypes = [u64, u64, u64, u32]
        L.or_fence_modulo_n.argtypes = [ctypes.c_void_p, u64, u64, u64, u32, ctypes.c_void_p]
        L.or_fence_modulo_n.restype = None
        L.or_fence_clamp.restype = u64
        L.or_fence_clamp.argtypes = [u64, u64, u64, u32]
        L.or_fence_clamp_n.argtypes = [ctypes.c_void_p, u64, u64, u64, u32, ctypes.c_void_p]
        L.or_fence_clamp_n.restype = None
        L.or_counted.restype = i32
        L.or_counted.argtypes = [P, u64, u32]
        L.or_check_ok.restype = i32
        L.or_check_ok.argtypes = [u64, u64, u64, u32]
        L.or_check_range.restype = i32
        L.or_check_range.argtypes = [u64, u64, u64, u64]
        L.or_resolve.restype = u64
        L.or_resolve.argtypes = [P, u64, u32, ctypes.POINTER(i32)]
        L.or_copy.argtypes = [P, u64, u64, u64]
        L.or_saxpy.argtypes = [P, f32, u64, u64, u64]
        L.or_gather.argtypes = [P, u64, u64, u64, u64, u32]
        L.or_scatter_add.argtypes = [P, u64, u64, u64, u64]
        L.or_stencil.argtypes = [P, u64, u64, u32, u32, u64, f32, f32]
        L.or_stencil_tma.argtypes = [P, u64, u64, u32, u32, u64, f32, f32]
        L.or_stencil_tma.restype = None
        L.or_desc_rows.restype = u64
        L.or_desc_rows.argtypes = [P, u64, u64, u64, u64, ctypes.POINTER(u64)]
        L.or_gemm.argtypes = [P, u64, u64, u64, u32, u32, u32, u64, u64, u64,
                              ctypes.POINTER(u32), u32]
        L.or_f32_to_bf16.restype = ctypes.c_uint16
        L.or_f32_to_bf16.argtypes = [f32]
        L.or_bf16_to_f32.restype = f32
        L.or_bf16_to_f32.argtypes = [ctypes.c_uint16]
        L.or_fence_mask_n.argtypes = [ctypes.c_void_p, u64, u64, u64, u32, ctypes.c_void_p]
        L.or_check_ok_n.argtypes = [ctypes.c_void_p, u64, u64, u64, u32, ctypes.c_void_p]
        for f in ("or_fence_mask_n", "or_check_ok_n", "or_copy", "or_saxpy", "or_gather", "or_scatter_add", "or_stencil", "or_gemm"):
            getattr(L, f).restype = None
        _lib = L
    return _lib


# --- scalar fence functions ---------------------------------------------------

def mask(size: int) -> int:
    return lib().or_mask(size)


def fence_modulo(a: int, base: int, size: int, w: int = 1) -> int:
    return lib().or_fence_modulo(a & (2**64 - 1), base, size, w)


def fence_clamp(a: int, base: int, size: int, w: int = 1) -> int:
    return lib().or_fence_clamp(a & (2**64 - 1), base, size, w)


def fence_mask(a: int, base: int, size: int, w: int = 1) -> int:
    return lib().or_fence_mask(a & (2**64 - 1), base, size, w)


def check_ok(a: int, base: int, size: int, w: int = 1) -> bool:
    return bool(lib().or_check_ok(a & (2**64 - 1), base, size, w))


def check_range(base: int, size: int, addr: int, length: int) -> bool:
    return bool(lib().or_check_range(base, size, addr & (2**64 - 1), length))


def fence_mask_n(a: np.ndarray, base: int, size: int, w: int = 1) -> np.ndarray:
    a = np.ascontiguousarray(a, dtype=np.uint64)
    out = np.empty_like(a)
    lib().or_fence_mask_n(a.ctypes.data, a.size, base, size, w, out.ctypes.data)
    return out


def fence_modulo_n(a: np.ndarray, base: int, size: int, w: int = 1) -> np.ndarray:
    a = np.ascontiguousarray(a, dtype=np.uint64)
    out = np.empty_like(a)
    lib().or_fence_modulo_n(a.ctypes.data, a.size, base, size, w, out.ctypes.data)
    return out


def fence_clamp_n(a: np.ndarray, base: int, size: int, w: int = 1) -> np.ndarray:
    a = np.ascontiguousarray(a, dtype=np.uint64)
    out = np.empty_like(a)
    lib().or_fence_clamp_n(a.ctypes.data, a.size, base, size, w, out.ctypes.data)
    return out


def check_ok_n(a: np.ndarray, base: int, size: int, w: int = 1) -> np.ndarray:
    a = np.ascontiguousarray(a, dtype=np.uint64)
    out = np.empty(a.shape, dtype=np.uint8)
    lib().or_check_ok_n(a.ctypes.data, a.size, base, size, w, out.ctypes.data)
    return out.astype(bool)


def f32_to_bf16(f: float) -> int:
    return lib().or_f32_to_bf16(f)


def bf16_to_f32(h: int) -> float:
    return lib().or_bf16_to_f32(h)


# --- simulated memory + launches -------------------------------------------------

@dataclass
class Counts:
    violations: int
    faults: int
    accesses: int


class Mem:
    """Simulated device memory: ``buf[k]`` stands for device address ``va + k``."""

    def __init__(self, va: int, nbytes: int | None = None, buf: np.ndarray | None = None):
        if buf is None:
            buf = np.zeros(nbytes, dtype=np.uint8)
        assert buf.dtype == np.uint8 and buf.flags["C_CONTIGUOUS"]
        self.va = va
        self.buf = buf

    def view(self, addr: int, dtype, count: int) -> np.ndarray:
        off = addr - self.va
        it = np.dtype(dtype).itemsize
        return self.buf[off:off + it * count].view(dtype)

    def write(self, addr: int, arr: np.ndarray) -> None:
        b = np.ascontiguousarray(arr).view(np.uint8).reshape(-1)
        off = addr - self.va
        self.buf[off:off + b.size] = b

    def ctx(self, base: int, size: int, mode) -> OrCtx:
        if isinstance(mode, str):
            mode = MODES[mode]
        return OrCtx(self.va, self.buf.size, self.buf.ctypes.data, base, size, mode, 0, 0, 0, 0)


def resolve(base: int, size: int, mode, a: int, w: int):
    """(address reached, ok) for one access in ``mode`` (no memory touched)."""
    if isinstance(mode, str):
        mode = MODES[mode]
    c = OrCtx(0, 0, None, base, size, mode, 0, 0, 0, 0)
    ok = ctypes.c_int(0)
    r = lib().or_resolve(ctypes.byref(c), a & (2**64 - 1), w, ctypes.byref(ok))
    return r, bool(ok.value)


def _run(fn, mem: Mem, base, size, mode, *args) -> Counts:
    c = mem.ctx(base, size, mode)
    fn(ctypes.byref(c), *args)
    return Counts(c.violations, c.faults, c.accesses)


def copy(mem, base, size, mode, dst, src, nbytes) -> Counts:
    return _run(lib().or_copy, mem, base, size, mode, dst, src, nbytes)


def saxpy(mem, base, size, mode, a, x, y, n) -> Counts:
    return _run(lib().or_saxpy, mem, base, size, mode, a, x, y, n)


def gather(mem, base, size, mode, out, table, idx, n, D=1) -> Counts:
    return _run(lib().or_gather, mem, base, size, mode, out, table, idx, n, D)


def scatter_add(mem, base, size, mode, table, idx, src, n) -> Counts:
    return _run(lib().or_scatter_add, mem, base, size, mode, table, idx, src, n)


def stencil(mem, base, size, mode, out, inp, H, W, pitch, c0, c1) -> Counts:
    return _run(lib().or_stencil, mem, base, size, mode, out, inp, H, W, pitch, c0, c1)


def stencil_tma(mem, base, size, mode, out, inp, H, W, pitch, c0, c1) -> Counts:
    return _run(lib().or_stencil_tma, mem, base, size, mode, out, inp, H, W, pitch, c0, c1)


def desc_rows(base, size, mode, p, rows, rowbytes, stride):
    if isinstance(mode, str):
        mode = MODES[mode]
    c = OrCtx(0, 0, None, base, size, mode, 0, 0, 0, 0)
    pf = ctypes.c_uint64(0)
    r = lib().or_desc_rows(ctypes.byref(c), p, rows, rowbytes, stride, ctypes.byref(pf))
    return r, pf.value


def gemm(mem, base, size, mode, C, A, B, M, N, K, lda, ldb, ldc, rows=None) -> Counts:
    if rows is None:
        rp, nr = None, 0
    else:
        r = np.ascontiguousarray(rows, dtype=np.uint32)
        rp, nr = r.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32)), r.size
    return _run(lib().or_gemm, mem, base, size, mode, C, A, B, M, N, K, lda, ldb, ldc, rp, nr)
