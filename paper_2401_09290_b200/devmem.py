"""Zero-copy torch views of raw device addresses (arena memory is not
allocated by torch).  Plumbing only: torch provides device memory, streams
and copies for tests and benchmarks, never the fenced computation.
"""
from __future__ import annotations

import torch

_TYPESTR = {torch.uint8: "|u1", torch.int8: "|i1", torch.int16: "<i2", torch.int32: "<i4",
            torch.int64: "<i8", torch.float32: "<f4", torch.float64: "<f8"}


class _CudaArray:
    def __init__(self, ptr: int, count: int, typestr: str):
        self.__cuda_array_interface__ = {"shape": (count,), "typestr": typestr, "data": (ptr, False),
                                         "version": 3, "strides": None, "stream": None}


def view(addr: int, count: int, dtype=torch.uint8, device: int = 0) -> torch.Tensor:
    """A 1-D tensor aliasing ``count`` elements of ``dtype`` at device address ``addr``."""
    if dtype == torch.bfloat16:
        return view(addr, count, torch.int16, device).view(torch.bfloat16)
    if count == 0:
        return torch.empty(0, dtype=dtype, device=f"cuda:{device}")
    with torch.cuda.device(device):
        return torch.as_tensor(_CudaArray(addr, count, _TYPESTR[dtype]), device=f"cuda:{device}")
