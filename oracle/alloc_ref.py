"""Naive bitmap partition allocator -- TEST INFRASTRUCTURE ONLY.

It exists to check the product's buddy allocator (paper_2401_09290_b200 csrc)
against the invariants SPEC.md:257-260 states, not its placement policy:
partitions are power-of-two sized (next_pow2(max(req, 4 KiB)), SPEC.md:217,
PAPER.md:246), aligned to their own size ("partitions to be in
the power of two"), pairwise disjoint, inside the arena,
and a request fails only when no aligned free slot of that size exists.

The arena is a bitmap of 4 KiB pages.  ``alloc`` scans the size-aligned slots
in ascending address order and takes the first one whose pages are all free.
"""
from __future__ import annotations

import numpy as np

PAGE = 4096
MIN_PARTITION = 4096


def next_pow2(n: int) -> int:
    p = 1
    while p < n:
        p *= 2
    return p


def partition_size(requested: int) -> int:
    return next_pow2(max(requested, MIN_PARTITION))


class BitmapArena:
    def __init__(self, base: int, size: int):
        assert size % PAGE == 0 and base % size == 0
        self.base, self.size = base, size
        self.used = np.zeros(size // PAGE, dtype=bool)
        self.live = {}  # base -> size

    def free_slot_exists(self, size: int) -> bool:
        return self._find(size) is not None

    def _find(self, size: int):
        if size > self.size:
            return None
        pages = size // PAGE
        for k in range(self.size // size):
            if not self.used[k * pages:(k + 1) * pages].any():
                return self.base + k * size
        return None

    def alloc(self, requested: int):
        size = partition_size(requested)
        b = self._find(size)
        if b is None:
            return None
        self.mark(b, size)
        return b, size

    def mark(self, b: int, size: int) -> None:
        """Record a partition placed by someone else (checks disjointness)."""
        lo = (b - self.base) // PAGE
        hi = lo + size // PAGE
        assert b % size == 0, "partition not aligned to its size"
        assert self.base <= b and b + size <= self.base + self.size, "partition outside arena"
        assert not self.used[lo:hi].any(), "partitions overlap"
        self.used[lo:hi] = True
        self.live[b] = size

    def free(self, b: int) -> None:
        size = self.live.pop(b)
        lo = (b - self.base) // PAGE
        self.used[lo:lo + size // PAGE] = False

    def free_bytes(self) -> int:
        return int((~self.used).sum()) * PAGE
