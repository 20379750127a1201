"""GPU parity of K4 v2, the radix-partitioned scatter-add (csrc/k_scatter.cu):
large scatters (>= 2^20 updates into partitions of >= 128 MiB) are applied
one 32 MiB partition slice at a time through a trusted scratch.  Every mode,
hoisted and per access, against the oracle's or_scatter_add over the WHOLE
partition byte for byte, violations exact, the victim partition unchanged.

Layout (256 MiB partition = 8 slices): table 64 MiB at 0, idx at 128 MiB,
src at 160 MiB, and the planted out-of-partition indices (5 %) wrap (mask /
modulo) into [192 MiB, 256 MiB), which nothing else touches (race-free,
SURVEY.md §8(c) O4); duplicates are heavy (u32 adds commute, reading A6).
The update count has a ragged tail (n % 4 = 3: the direct kernel's part).
"""
import numpy as np
import pytest

import oracle
import synth
from tests.gpu_util import download, first_diff, upload

pytestmark = pytest.mark.gpu

MiB = 1 << 20
PART = 256 * MiB
IDX, SRC, PAT_LO = 128 * MiB, 160 * MiB, 192 * MiB
TABLE_WORDS = (64 * MiB) // 4


@pytest.mark.parametrize("mode", ["none", "mask", "check", "modulo", "maskcount", "clamp",
                                  "check+pa", "clamp+pa", "maskcount+pa"])
def test_bucketed_scatter_matches_oracle(arenas, mode):
    a = arenas(2 * PART)
    victim = a.partition_alloc(PART)
    p = a.partition_alloc(PART)
    rng = synth.rng_for(8800)
    n = (1 << 21) + 3
    j = rng.integers(0, TABLE_WORDS, n, dtype=np.int64)
    hot = rng.random(n) < 0.25                         # a quarter of the updates hit 64 hot words
    j[hot] = rng.integers(0, 64, int(hot.sum()))
    base_mode = mode.split("+")[0]
    planted = 0
    if base_mode != "none":
        planted = synth.planted_count(0.05, n)
        pos = synth.planted_positions(rng, n, planted)
        if base_mode == "clamp":                        # clamped adds pile up on the two edge words
            j[pos] = np.where(rng.random(planted) < 0.5, -(1 << 31), (1 << 31) - 1)
        else:
            j[pos] = synth.oob_indices(rng, planted, PART // 4, PAT_LO // 4, PART // 4)
    upload(victim.base, synth.random_bytes(rng, 16 * MiB))
    upload(p.base, synth.random_bytes(rng, 64 * MiB))
    upload(p.base + IDX, j.astype(np.int32))
    upload(p.base + SRC, synth.uniform_u32(rng, n))
    before = download(a.base, a.size)
    a.stats_reset()
    a.scatter(p.id, mode, p.base, p.base + IDX, p.base + SRC, n)
    st = a.stats(p.id)
    after = download(a.base, a.size)
    lo = p.base - a.base
    mem = oracle.Mem(p.base, buf=before[lo:lo + PART].copy())
    c = oracle.scatter_add(mem, p.base, p.size, base_mode, p.base, p.base + IDX, p.base + SRC, n)
    got = after[lo:lo + PART]
    assert np.array_equal(got, mem.buf), first_diff(got, mem.buf)
    assert np.array_equal(after[:lo], before[:lo]), "the victim partition was modified"
    assert c.faults == 0
    assert st["violations"] == c.violations
    assert c.violations == (planted if base_mode in ("check", "maskcount", "clamp") else 0)
    assert a.device_flags() == 0


def test_bucketed_scatter_in_a_captured_graph(arenas):
    """The scratch is allocated stream-ordered (cudaMallocAsync), so the
    bucketed scatter can be captured into a graph (gd_graph_create) and
    replayed; three replays add three times."""
    from paper_2401_09290_b200 import guardian as g
    a = arenas(PART)
    p = a.partition_alloc(PART)
    rng = synth.rng_for(8801)
    n = 1 << 20
    j = rng.integers(0, TABLE_WORDS, n, dtype=np.int64).astype(np.int32)
    s = synth.uniform_u32(rng, n)
    upload(p.base + IDX, j)
    upload(p.base + SRC, s)
    item = g.work(p.id, g.GD_KIND_SCATTER, "check", ptr=(p.base, p.base + IDX, p.base + SRC), u64=(n,))
    gr = a.graph([item], n_streams=1)
    for _ in range(3):
        gr.launch()
    got = download(p.base, 64 * MiB).view(np.uint32)
    want = np.zeros(TABLE_WORDS, np.uint64)
    np.add.at(want, j.astype(np.int64), 3 * s.astype(np.uint64))
    assert np.array_equal(got, (want & 0xFFFFFFFF).astype(np.uint32))
    gr.close()
