"""Thin ctypes binding of libguardian.so (include/guardian.h).

Argument marshalling only: every step of the fenced path runs in the
library's sm_100a kernels.  There is no fallback -- if libguardian.so is
missing or fails to load, importing this module raises.

Names follow the C ABI (``gd_arena_create`` ...).  ``Arena`` is a small
convenience wrapper used by the tests and ``bench.py``; it raises
``GuardianError`` for any non-OK status.
"""
from __future__ import annotations

import ctypes
import os

_PKG = os.path.dirname(os.path.abspath(__file__))
# GD_LIB: a development build of the same library (tools/ A/B probes only)
LIB_PATH = os.environ.get("GD_LIB") or os.path.join(_PKG, "libguardian.so")

GD_OK = 0
STATUS = ["GD_OK", "GD_ERR_INVALID_ARG", "GD_ERR_NOT_POW2", "GD_ERR_DEVICE_OOM", "GD_ERR_PARTITION_OOM",
          "GD_ERR_UNKNOWN_PARTITION", "GD_ERR_UNKNOWN_ALLOC", "GD_ERR_ALIGN", "GD_ERR_OOB_RANGE",
          "GD_ERR_UNSUPPORTED", "GD_ERR_CUDA"]
(GD_ERR_INVALID_ARG, GD_ERR_NOT_POW2, GD_ERR_DEVICE_OOM, GD_ERR_PARTITION_OOM, GD_ERR_UNKNOWN_PARTITION,
 GD_ERR_UNKNOWN_ALLOC, GD_ERR_ALIGN, GD_ERR_OOB_RANGE, GD_ERR_UNSUPPORTED, GD_ERR_CUDA) = range(1, 11)
GD_MODE_NONE, GD_MODE_MASK, GD_MODE_CHECK = 0, 1, 2
GD_MODE_MODULO, GD_MODE_MASK_COUNT, GD_MODE_CLAMP = 3, 4, 5
GD_FENCE_PER_ACCESS = 0x100       # OR-ed into a mode: fence every access (no tile-level range test)
MODES = {"none": GD_MODE_NONE, "mask": GD_MODE_MASK, "check": GD_MODE_CHECK, "modulo": GD_MODE_MODULO,
         "maskcount": GD_MODE_MASK_COUNT, "clamp": GD_MODE_CLAMP}
GD_POLICY_ROUND_ROBIN, GD_POLICY_NO_TENSOR_RANDOM, GD_POLICY_MEMORY_LANE = 0, 1, 2
POLICIES = {"round_robin": GD_POLICY_ROUND_ROBIN, "no_tensor_random": GD_POLICY_NO_TENSOR_RANDOM,
            "memory_lane": GD_POLICY_MEMORY_LANE}
GD_PART_POW2 = 1
(GD_KIND_COPY, GD_KIND_SAXPY, GD_KIND_GATHER, GD_KIND_SCATTER, GD_KIND_STENCIL, GD_KIND_GEMM) = range(6)
GD_NUM_KINDS = 6
GD_MAX_TENANTS = 64
GD_ALL_TENANTS = 0xFFFFFFFF
KIND_NAMES = ["copy", "saxpy", "gather", "scatter", "stencil", "gemm"]

EXPORTED = [
    "gd_arena_create", "gd_arena_wrap", "gd_arena_destroy", "gd_arena_info", "gd_arena_set_native_when_solo",
    "gd_partition_alloc", "gd_partition_alloc_exact", "gd_partition_free", "gd_partition_get", "gd_malloc", "gd_free",
    "gd_check_range", "gd_memcpy_h2d", "gd_memcpy_d2h", "gd_memcpy_d2d", "gd_partition_fill",
    "gd_launch_fenced_copy", "gd_launch_fenced_saxpy", "gd_launch_fenced_gather",
    "gd_launch_fenced_scatter", "gd_launch_fenced_stencil", "gd_launch_fenced_stencil_tma", "gd_launch_fenced_gemm",
    "gd_schedule_round_robin", "gd_launcher_run", "gd_launcher_run_policy",
    "gd_stats", "gd_stats_reset", "gd_stats_device_ptr", "gd_status_str", "gd_last_cuda_error", "gd_version",
    "gd_device_flags", "gd_graph_create", "gd_graph_launch", "gd_graph_destroy",
]


class gd_partition_info(ctypes.Structure):
    _fields_ = [("id", ctypes.c_uint32), ("flags", ctypes.c_uint32), ("base", ctypes.c_uint64),
                ("size", ctypes.c_uint64), ("mask", ctypes.c_uint64), ("end", ctypes.c_uint64)]


class gd_stats_t(ctypes.Structure):
    _fields_ = [("violations", ctypes.c_uint64), ("launches", ctypes.c_uint64), ("bytes", ctypes.c_uint64),
                ("flops", ctypes.c_uint64), ("violations_by_kind", ctypes.c_uint64 * GD_NUM_KINDS),
                ("launches_by_kind", ctypes.c_uint64 * GD_NUM_KINDS)]


class gd_work(ctypes.Structure):
    _fields_ = [("tenant", ctypes.c_uint32), ("kind", ctypes.c_uint32), ("mode", ctypes.c_uint32),
                ("u32", ctypes.c_uint32 * 3), ("ptr", ctypes.c_uint64 * 3), ("u64", ctypes.c_uint64 * 3),
                ("f32", ctypes.c_float * 2)]


class GuardianError(RuntimeError):
    def __init__(self, fn: str, status: int):
        self.status = status
        name = STATUS[status] if 0 <= status < len(STATUS) else str(status)
        extra = f" (cuda error {_lib.gd_last_cuda_error()})" if status == GD_ERR_CUDA else ""
        super().__init__(f"{fn} -> {name}{extra}")


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'` "
                          "(there is no CPU fallback)")
    L = ctypes.CDLL(LIB_PATH)
    u32, u64, f32, vp, i32 = ctypes.c_uint32, ctypes.c_uint64, ctypes.c_float, ctypes.c_void_p, ctypes.c_int
    A = vp                           # gd_arena*
    P = ctypes.POINTER
    sig = {
        "gd_arena_create": [i32, u64, u32, P(vp)],
        "gd_arena_wrap": [i32, u64, u64, P(vp)],
        "gd_arena_set_native_when_solo": [A, i32],
        "gd_arena_destroy": [A],
        "gd_arena_info": [A, P(u64), P(u64), P(i32)],
        "gd_partition_alloc": [A, u64, P(gd_partition_info)],
        "gd_partition_alloc_exact": [A, u64, P(gd_partition_info)],
        "gd_partition_free": [A, u32],
        "gd_partition_get": [A, u32, P(gd_partition_info)],
        "gd_malloc": [A, u32, u64, P(u64)],
        "gd_free": [A, u32, u64],
        "gd_check_range": [A, u32, u64, u64, P(i32)],
        "gd_memcpy_h2d": [A, u32, u64, vp, u64, vp],
        "gd_memcpy_d2h": [A, u32, vp, u64, u64, vp],
        "gd_memcpy_d2d": [A, u32, u64, u64, u64, vp],
        "gd_partition_fill": [A, u32, u32, u64, u64, vp],
        "gd_launch_fenced_copy": [A, u32, i32, u64, u64, u64, vp],
        "gd_launch_fenced_saxpy": [A, u32, i32, f32, u64, u64, u64, vp],
        "gd_launch_fenced_gather": [A, u32, i32, u64, u64, u64, u64, u32, vp],
        "gd_launch_fenced_scatter": [A, u32, i32, u64, u64, u64, u64, vp],
        "gd_launch_fenced_stencil": [A, u32, i32, u64, u64, u32, u32, u64, f32, f32, vp],
        "gd_launch_fenced_stencil_tma": [A, u32, i32, u64, u64, u32, u32, u64, f32, f32, vp],
        "gd_launch_fenced_gemm": [A, u32, i32, u64, u64, u64, u32, u32, u32, u64, u64, u64, vp],
        "gd_schedule_round_robin": [P(gd_work), u32, P(u32)],
        "gd_launcher_run": [A, P(gd_work), u32, P(vp), u32, P(u32)],
        "gd_launcher_run_policy": [A, P(gd_work), u32, P(vp), u32, u32, P(u32)],
        "gd_stats": [A, u32, P(gd_stats_t)],
        "gd_stats_reset": [A, u32],
        "gd_stats_device_ptr": [A, P(u64)],
        "gd_device_flags": [A, P(u32)],
        "gd_graph_create": [A, P(gd_work), u32, u32, P(vp)],
        "gd_graph_launch": [vp, vp],
        "gd_graph_destroy": [vp],
    }
    for name, args in sig.items():
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = ctypes.c_int
    L.gd_status_str.argtypes = [ctypes.c_int]
    L.gd_status_str.restype = ctypes.c_char_p
    L.gd_last_cuda_error.argtypes = []
    L.gd_last_cuda_error.restype = ctypes.c_int
    L.gd_version.argtypes = []
    L.gd_version.restype = ctypes.c_char_p
    return L


_lib = _load()


def lib():
    return _lib


def _chk(fn: str, st: int) -> None:
    if st != GD_OK:
        raise GuardianError(fn, st)


def _stream(s) -> int | None:
    """Accept None, an int handle, or a torch.cuda.Stream."""
    if s is None:
        return None
    if isinstance(s, int):
        return s
    return s.cuda_stream


def _mode(m) -> int:
    """A mode name ("check"), optionally with the per-access suffix
    ("check+pa" = GD_MODE_CHECK | GD_FENCE_PER_ACCESS), or an int."""
    if isinstance(m, str):
        name, _, flag = m.partition("+")
        if flag not in ("", "pa"):
            raise ValueError(f"unknown mode suffix in {m!r}")
        return MODES[name] | (GD_FENCE_PER_ACCESS if flag else 0)
    return int(m)


# --- the C names, one-to-one (status codes returned) -------------------------

def gd_arena_create(device: int, arena_bytes: int, flags: int = 0):
    p = ctypes.c_void_p()
    return _lib.gd_arena_create(device, arena_bytes, flags, ctypes.byref(p)), p


def gd_arena_wrap(device: int, dev_ptr: int, nbytes: int):
    p = ctypes.c_void_p()
    return _lib.gd_arena_wrap(device, dev_ptr, nbytes, ctypes.byref(p)), p


def gd_schedule_round_robin(items):
    arr = (gd_work * len(items))(*items)
    out = (ctypes.c_uint32 * max(1, len(items)))()
    st = _lib.gd_schedule_round_robin(arr, len(items), out)
    return st, list(out)[:len(items)]


def work(tenant, kind, mode, ptr=(), u64=(), u32=(), f32=()) -> gd_work:
    w = gd_work()
    w.tenant, w.kind, w.mode = tenant, kind, _mode(mode)
    for i, v in enumerate(ptr):
        w.ptr[i] = v
    for i, v in enumerate(u64):
        w.u64[i] = v
    for i, v in enumerate(u32):
        w.u32[i] = v
    for i, v in enumerate(f32):
        w.f32[i] = v
    return w


# --- convenience wrapper ------------------------------------------------------

class Partition:
    def __init__(self, info: gd_partition_info):
        self.id, self.base, self.size = info.id, info.base, info.size
        self.mask, self.end = info.mask, info.end
        self.pow2 = bool(info.flags & GD_PART_POW2)

    def __repr__(self):
        return f"Partition(id={self.id}, base={self.base:#x}, size={self.size:#x})"


class Graph:
    """A captured multi-tenant step (gd_graph)."""

    def __init__(self, h):
        self._h = h

    def launch(self, stream=None) -> None:
        _chk("gd_graph_launch", _lib.gd_graph_launch(self._h, _stream(stream)))

    def close(self) -> None:
        if self._h is not None and self._h.value:
            _chk("gd_graph_destroy", _lib.gd_graph_destroy(self._h))
        self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Arena:
    """Owns a gd_arena.  ``Arena(device, nbytes)`` reserves a VMM arena;
    ``Arena.wrap(device, ptr, nbytes)`` uses caller-owned memory
    (device < 0: virtual, bookkeeping only)."""

    def __init__(self, device: int = 0, nbytes: int = 1 << 20, _handle=None):
        if _handle is None:
            st, h = gd_arena_create(device, nbytes, 0)
            _chk("gd_arena_create", st)
        else:
            h = _handle
        self._h = h
        b, s, d = ctypes.c_uint64(), ctypes.c_uint64(), ctypes.c_int()
        _chk("gd_arena_info", _lib.gd_arena_info(h, ctypes.byref(b), ctypes.byref(s), ctypes.byref(d)))
        self.base, self.size, self.device = b.value, s.value, d.value

    @classmethod
    def wrap(cls, device: int, dev_ptr: int, nbytes: int) -> "Arena":
        st, h = gd_arena_wrap(device, dev_ptr, nbytes)
        _chk("gd_arena_wrap", st)
        return cls(_handle=h)

    @property
    def handle(self):
        return self._h

    def set_native_when_solo(self, on: bool) -> None:
        """a tenant alone runs the native (unfenced) kernel."""
        _chk("gd_arena_set_native_when_solo", _lib.gd_arena_set_native_when_solo(self._h, int(bool(on))))

    def close(self):
        if self._h is not None and self._h.value:
            _chk("gd_arena_destroy", _lib.gd_arena_destroy(self._h))
        self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    # partitions ---------------------------------------------------------
    def partition_alloc_exact(self, requested: int) -> Partition:
        info = gd_partition_info()
        _chk("gd_partition_alloc_exact", _lib.gd_partition_alloc_exact(self._h, requested, ctypes.byref(info)))
        return Partition(info)

    def partition_alloc(self, requested: int) -> Partition:
        info = gd_partition_info()
        _chk("gd_partition_alloc", _lib.gd_partition_alloc(self._h, requested, ctypes.byref(info)))
        return Partition(info)

    def partition_free(self, pid: int) -> None:
        _chk("gd_partition_free", _lib.gd_partition_free(self._h, pid))

    def partition_get(self, pid: int) -> Partition:
        info = gd_partition_info()
        _chk("gd_partition_get", _lib.gd_partition_get(self._h, pid, ctypes.byref(info)))
        return Partition(info)

    def malloc(self, pid: int, nbytes: int) -> int:
        a = ctypes.c_uint64()
        _chk("gd_malloc", _lib.gd_malloc(self._h, pid, nbytes, ctypes.byref(a)))
        return a.value

    def free(self, pid: int, addr: int) -> None:
        _chk("gd_free", _lib.gd_free(self._h, pid, addr))

    def check_range(self, pid: int, addr: int, length: int) -> bool:
        ok = ctypes.c_int()
        _chk("gd_check_range", _lib.gd_check_range(self._h, pid, addr, length, ctypes.byref(ok)))
        return bool(ok.value)

    def memcpy_h2d(self, pid: int, dst: int, host_ptr: int, n: int, stream=None) -> None:
        _chk("gd_memcpy_h2d", _lib.gd_memcpy_h2d(self._h, pid, dst, host_ptr, n, _stream(stream)))

    def memcpy_d2d(self, pid: int, dst: int, src: int, n: int, stream=None) -> None:
        _chk("gd_memcpy_d2d", _lib.gd_memcpy_d2d(self._h, pid, dst, src, n, _stream(stream)))

    def memcpy_d2h(self, pid: int, host_ptr: int, src: int, n: int, stream=None) -> None:
        _chk("gd_memcpy_d2h", _lib.gd_memcpy_d2h(self._h, pid, host_ptr, src, n, _stream(stream)))

    def fill(self, pid: int, pattern: int, offset: int, nbytes: int, stream=None) -> None:
        _chk("gd_partition_fill", _lib.gd_partition_fill(self._h, pid, pattern, offset, nbytes, _stream(stream)))

    # fenced launches ----------------------------------------------------
    def copy(self, pid, mode, dst, src, nbytes, stream=None):
        _chk("gd_launch_fenced_copy",
             _lib.gd_launch_fenced_copy(self._h, pid, _mode(mode), dst, src, nbytes, _stream(stream)))

    def saxpy(self, pid, mode, alpha, x, y, n, stream=None):
        _chk("gd_launch_fenced_saxpy",
             _lib.gd_launch_fenced_saxpy(self._h, pid, _mode(mode), alpha, x, y, n, _stream(stream)))

    def gather(self, pid, mode, out, table, idx, n, row_elems=1, stream=None):
        _chk("gd_launch_fenced_gather",
             _lib.gd_launch_fenced_gather(self._h, pid, _mode(mode), out, table, idx, n, row_elems,
                                          _stream(stream)))

    def scatter(self, pid, mode, table, idx, src, n, stream=None):
        _chk("gd_launch_fenced_scatter",
             _lib.gd_launch_fenced_scatter(self._h, pid, _mode(mode), table, idx, src, n, _stream(stream)))

    def stencil(self, pid, mode, out, inp, H, W, pitch, c0, c1, stream=None):
        _chk("gd_launch_fenced_stencil",
             _lib.gd_launch_fenced_stencil(self._h, pid, _mode(mode), out, inp, H, W, pitch, c0, c1,
                                           _stream(stream)))

    def stencil_tma(self, pid, mode, out, inp, H, W, pitch, c0, c1, stream=None):
        """K5 v2: both operands TMA-staged and descriptor-fenced."""
        _chk("gd_launch_fenced_stencil_tma",
             _lib.gd_launch_fenced_stencil_tma(self._h, pid, _mode(mode), out, inp, H, W, pitch, c0, c1,
                                               _stream(stream)))

    def gemm(self, pid, mode, C, A, B, M, N, K, lda, ldb, ldc, stream=None):
        _chk("gd_launch_fenced_gemm",
             _lib.gd_launch_fenced_gemm(self._h, pid, _mode(mode), C, A, B, M, N, K, lda, ldb, ldc,
                                        _stream(stream)))

    def graph(self, items, n_streams: int) -> "Graph":
        """Capture one launcher step of `items` into a CUDA graph."""
        arr = (gd_work * len(items))(*items)
        h = ctypes.c_void_p()
        _chk("gd_graph_create", _lib.gd_graph_create(self._h, arr, len(items), n_streams, ctypes.byref(h)))
        return Graph(h)

    def launcher_run(self, items, streams, policy="round_robin"):
        """gd_launcher_run_policy: policy "round_robin" (the paper's launcher)
        , "no_tensor_random" (GEMMs never overlap gathers / scatters) or
        "memory_lane" (memory-bound kernels serialised, GEMMs overlap them)."""
        arr = (gd_work * len(items))(*items)
        sarr = (ctypes.c_void_p * len(streams))(*[_stream(s) for s in streams])
        order = (ctypes.c_uint32 * max(1, len(items)))()
        pol = POLICIES[policy] if isinstance(policy, str) else int(policy)
        _chk("gd_launcher_run_policy",
             _lib.gd_launcher_run_policy(self._h, arr, len(items), sarr, len(streams), pol, order))
        return list(order)[:len(items)]

    # statistics -----------------------------------------------------------
    def stats(self, pid: int = GD_ALL_TENANTS) -> dict:
        s = gd_stats_t()
        _chk("gd_stats", _lib.gd_stats(self._h, pid, ctypes.byref(s)))
        return {"violations": s.violations, "launches": s.launches, "bytes": s.bytes, "flops": s.flops,
                "violations_by_kind": dict(zip(KIND_NAMES, list(s.violations_by_kind))),
                "launches_by_kind": dict(zip(KIND_NAMES, list(s.launches_by_kind)))}

    def stats_reset(self, pid: int = GD_ALL_TENANTS) -> None:
        _chk("gd_stats_reset", _lib.gd_stats_reset(self._h, pid))

    def device_flags(self) -> int:
        f = ctypes.c_uint32()
        _chk("gd_device_flags", _lib.gd_device_flags(self._h, ctypes.byref(f)))
        return f.value

    def stats_device_ptr(self) -> int:
        p = ctypes.c_uint64()
        _chk("gd_stats_device_ptr", _lib.gd_stats_device_ptr(self._h, ctypes.byref(p)))
        return p.value


def version() -> str:
    return _lib.gd_version().decode()
