"""Helpers for the GPU parity tests: move bytes between NumPy and raw device
addresses (torch does the copies; the fenced work runs in libguardian.so)."""
import numpy as np
import torch

from paper_2401_09290_b200 import devmem


def upload(addr: int, arr: np.ndarray) -> None:
    b = np.ascontiguousarray(arr).view(np.uint8).reshape(-1)
    devmem.view(addr, b.size, torch.uint8).copy_(torch.from_numpy(b))


def download(addr: int, nbytes: int) -> np.ndarray:
    torch.cuda.synchronize()
    return devmem.view(addr, nbytes, torch.uint8).cpu().numpy()


def first_diff(a: np.ndarray, b: np.ndarray) -> str:
    d = np.nonzero(a != b)[0]
    if d.size == 0:
        return "identical"
    return f"{d.size} bytes differ, first at offset {d[0]:#x}: got {a[d[0]]} expected {b[d[0]]}"
