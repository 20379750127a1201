"""B200-native (sm_100a) per-access address fencing after Guardian
(arXiv 2401.09290): partition manager, C-ABI library libguardian.so with
fenced copy / saxpy / gather / scatter / stencil / GEMM kernels, multi-tenant
launcher.  See DESIGN.md.

``from paper_2401_09290_b200 import guardian`` loads libguardian.so (and
fails loudly if it is not built: there is no CPU fallback).
"""
__all__ = ["guardian", "devmem", "build"]
