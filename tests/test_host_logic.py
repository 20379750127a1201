"""Host-side logic of libguardian.so, on CPU (no GPU calls): the C ABI loads
and exports every symbol include/guardian.h declares; the partition manager
(virtual arena) keeps the SPEC invariants against the naive bitmap allocator;
the sub-allocator, host-transfer range check, launch validation and the
round-robin schedule behave as specified."""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

import oracle
from oracle.alloc_ref import BitmapArena, partition_size
from paper_2401_09290_b200 import guardian as g

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HDR = os.path.join(ROOT, "include", "guardian.h")
DEV_BASE = 0x7FA2C0000000


def declared_symbols():
    src = open(HDR).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(gd_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    names = declared_symbols()
    assert len(names) >= 25
    lib = ctypes.CDLL(g.LIB_PATH)
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    out = subprocess.run(["nm", "-D", "--defined-only", g.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (gd_[a-z0-9_]+)", out))
    assert set(names) <= exported
    assert set(g.EXPORTED) == set(names), set(g.EXPORTED) ^ set(names)


def test_library_is_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", g.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_status_strings():
    for i, name in enumerate(g.STATUS):
        assert g.lib().gd_status_str(i).decode() == name


def virtual(size=32 << 20, base=DEV_BASE):
    return g.Arena.wrap(-1, base, size)


def test_spec_partition_examples():
    """SPEC.md:219-221 (create_partition examples)."""
    import json
    ex = json.load(open(os.path.join(ROOT, "tests", "golden", "paper_fence_examples.json")))["partition_placement"]
    a = virtual(ex["device_size"], int(ex["device_base"], 16))
    got = []
    for req in ex["requests"]:
        try:
            got.append(a.partition_alloc(req).base)
        except g.GuardianError as e:
            assert e.status == g.GD_ERR_DEVICE_OOM
            got.append(None)
    assert got == [None if x is None else int(x, 16) for x in ex["expect"]]
    b = virtual()
    p = b.partition_alloc(1)
    assert p.size == 4096 and p.mask == 0xFFF and p.end == p.base + 4096


def test_equal_requests_are_consecutive():
    """P13: equal-size requests in a fresh arena give base_t = arena + t*size."""
    a = virtual(1 << 20)
    parts = [a.partition_alloc(256 << 10) for _ in range(4)]
    assert [p.base for p in parts] == [DEV_BASE + t * (256 << 10) for t in range(4)]
    with pytest.raises(g.GuardianError) as e:
        a.partition_alloc(1)
    assert e.value.status == g.GD_ERR_DEVICE_OOM


def test_free_and_recreate_same_base():
    a = virtual()
    p = a.partition_alloc(5 << 20)
    a.partition_free(p.id)
    q = a.partition_alloc(5 << 20)
    assert q.base == p.base and q.size == 8 << 20
    with pytest.raises(g.GuardianError) as e:
        a.partition_free(63)
    assert e.value.status == g.GD_ERR_UNKNOWN_PARTITION


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_buddy_fuzz_against_bitmap(seed):
    """aligned, disjoint, inside, conserving; a request
    fails iff no aligned free slot of its size exists."""
    size = 1 << 24
    a = virtual(size)
    ref = BitmapArena(DEV_BASE, size)
    rng = np.random.Generator(np.random.PCG64(seed))
    live = {}
    for _ in range(1500):
        if live and (rng.random() < 0.45 or len(live) >= 60):
            pid = int(rng.choice(list(live)))
            a.partition_free(pid)
            ref.free(live.pop(pid))
        else:
            req = int(2 ** rng.uniform(0, 23.5))
            exists = ref.free_slot_exists(partition_size(req))
            try:
                p = a.partition_alloc(req)
            except g.GuardianError as e:
                assert e.status == g.GD_ERR_DEVICE_OOM and not exists
                continue
            assert exists
            assert p.size == partition_size(req) and p.base % p.size == 0
            ref.mark(p.base, p.size)                   # asserts aligned, inside, disjoint
            live[p.id] = p.base
        assert ref.free_bytes() + sum(ref.live.values()) == size


def test_suballocator_spec_examples():
    a = virtual()
    p = a.partition_alloc(16 << 20)
    x = a.malloc(p.id, 1024)
    assert x == p.base                                      # first fit from offset 0
    with pytest.raises(g.GuardianError) as e:
        a.malloc(p.id, 0)
    assert e.value.status == g.GD_ERR_INVALID_ARG
    with pytest.raises(g.GuardianError) as e:
        a.free(p.id, x + 8)
    assert e.value.status == g.GD_ERR_UNKNOWN_ALLOC
    a.free(p.id, x)
    assert a.malloc(p.id, 16 << 20) == p.base               # back to one full extent
    q = a.partition_alloc(16 << 10)
    n = 0
    while True:
        try:
            addr = a.malloc(q.id, 256)
        except g.GuardianError as e:
            assert e.status == g.GD_ERR_PARTITION_OOM
            break
        assert addr % 256 == 0 and q.base <= addr < q.end
        n += 1
    assert n * 256 == q.size


def test_suballocator_fuzz_tiling():
    a = virtual()
    p = a.partition_alloc(1 << 20)
    rng = np.random.Generator(np.random.PCG64(9))
    live = {}
    for _ in range(3000):
        if live and rng.random() < 0.5:
            addr = int(rng.choice(list(live)))
            a.free(p.id, addr)
            live.pop(addr)
        else:
            n = int(rng.integers(1, 20000))
            try:
                addr = a.malloc(p.id, n)
            except g.GuardianError as e:
                assert e.status == g.GD_ERR_PARTITION_OOM
                continue
            assert addr % 256 == 0 and p.base <= addr and addr + n <= p.end
            for b, m in live.items():
                assert addr + n <= b or b + m <= addr
            live[addr] = n


def test_check_range_matches_oracle():
    a = virtual()
    p = a.partition_alloc(16 << 20)
    rng = np.random.Generator(np.random.PCG64(5))
    cases = [(p.base, 0), (p.end, 0), (p.end + 1, 0), (p.base - 1, 1), (p.end - 1, 1), (p.end - 1, 2),
             (2**64 - 8, 16), (p.base, p.size), (p.base, p.size + 1)]
    for _ in range(2000):
        cases.append((int(rng.integers(p.base - 4096, p.end + 4096)), int(rng.integers(0, 1 << 21))))
    for addr, n in cases:
        assert a.check_range(p.id, addr, n) == oracle.check_range(p.base, p.size, addr, n), (addr, n)


def test_launch_validation_on_virtual_arena():
    a = virtual()
    p = a.partition_alloc(1 << 20)
    with pytest.raises(g.GuardianError) as e:
        a.copy(p.id, "mask", p.base + 8, p.base, 64)
    assert e.value.status == g.GD_ERR_ALIGN
    with pytest.raises(g.GuardianError) as e:
        a.copy(p.id, 7, p.base, p.base, 64)
    assert e.value.status == g.GD_ERR_INVALID_ARG
    with pytest.raises(g.GuardianError) as e:
        a.gather(9, "mask", p.base, p.base, p.base, 4)
    assert e.value.status == g.GD_ERR_UNKNOWN_PARTITION
    with pytest.raises(g.GuardianError) as e:
        a.gemm(p.id, "mask", p.base, p.base, p.base, 128, 128, 100, 128, 128, 128)
    assert e.value.status == g.GD_ERR_UNSUPPORTED                         # K % 64
    with pytest.raises(g.GuardianError) as e:
        a.stencil(p.id, "mask", p.base, p.base, 10, 10, 9, 0.5, 0.125)
    assert e.value.status in (g.GD_ERR_ALIGN, g.GD_ERR_INVALID_ARG)
    a.copy(p.id, "mask", p.base, p.base, 0)                               # n = 0: OK, no work
    with pytest.raises(g.GuardianError) as e:
        a.copy(p.id, "mask", p.base, p.base + 16, 64)                     # valid, but no device
    assert e.value.status == g.GD_ERR_UNSUPPORTED
    # size limits (every grid below 2^31 CTAs), refused before anything runs
    for call in (lambda: a.copy(p.id, "mask", p.base, p.base, (1 << 44) + 16),
                 lambda: a.saxpy(p.id, "mask", 1.0, p.base, p.base, (1 << 42) + 4),
                 lambda: a.gather(p.id, "mask", p.base, p.base, p.base, (1 << 40) + 4, 8),
                 lambda: a.gather(p.id, "mask", p.base, p.base + 4, p.base, (1 << 40) + 1, 2),   # flat words: 2^41 + 2
                 lambda: a.scatter(p.id, "mask", p.base, p.base, p.base, (1 << 42) + 4)):
        with pytest.raises(g.GuardianError) as e:
            call()
        assert e.value.status == g.GD_ERR_INVALID_ARG
    with pytest.raises(g.GuardianError) as e:
        a.stencil(p.id, "mask", p.base, p.base, (1 << 19) + 1, 8, 8, 0.5, 0.125)
    assert e.value.status == g.GD_ERR_UNSUPPORTED
    with pytest.raises(g.GuardianError) as e:                          # the TMA stencil takes it
        a.stencil_tma(p.id, "mask", p.base, p.base, (1 << 19) + 1, 8, 8, 0.5, 0.125)
    assert e.value.status == g.GD_ERR_UNSUPPORTED                         # (valid; no device here)


def test_per_access_flag_validation():
    """GD_FENCE_PER_ACCESS is a flag OR-ed into the mode of any launch
    (include/guardian.h): accepted with every mode, any other bit above the
    mode byte or a mode past CLAMP is INVALID_ARG, before anything runs."""
    a = virtual()
    p = a.partition_alloc(1 << 20)
    for m in ("none", "mask", "check", "modulo", "maskcount", "clamp"):
        with pytest.raises(g.GuardianError) as e:                       # valid; no device here
            a.copy(p.id, m + "+pa", p.base, p.base + 16, 64)
        assert e.value.status == g.GD_ERR_UNSUPPORTED
        assert g._mode(m + "+pa") == g.MODES[m] | g.GD_FENCE_PER_ACCESS
    for bad in (g.GD_MODE_CHECK | 0x200, g.GD_MODE_CHECK | 0x10000, 6 | g.GD_FENCE_PER_ACCESS, 0xFF):
        with pytest.raises(g.GuardianError) as e:
            a.copy(p.id, bad, p.base, p.base + 16, 64)
        assert e.value.status == g.GD_ERR_INVALID_ARG
    with pytest.raises(ValueError):
        g._mode("check+xx")
    items = [g.work(p.id, g.GD_KIND_COPY, "check+pa", ptr=(p.base, p.base + 64), u64=(64,)),
             g.work(p.id, g.GD_KIND_COPY, g.GD_MODE_MASK | 0x400, ptr=(p.base, p.base + 64), u64=(64,))]
    with pytest.raises(g.GuardianError) as e:                            # launcher: bad flag found first
        a.launcher_run(items, [None])
    assert e.value.status == g.GD_ERR_INVALID_ARG


def test_arena_wrap_errors():
    st, _ = g.gd_arena_wrap(-1, DEV_BASE, 3 << 20)
    assert st == g.GD_ERR_NOT_POW2
    st, _ = g.gd_arena_wrap(-1, DEV_BASE + 4096, 1 << 20)
    assert st == g.GD_ERR_ALIGN


def _items(tenants):
    return [g.work(t, g.GD_KIND_COPY, "mask", u64=(16 * i,)) for i, t in enumerate(tenants)]


def test_round_robin_spec_example():
    """queued a1, a2, b1 -> issue a1, b1, a2."""
    st, order = g.gd_schedule_round_robin(_items([0, 0, 1]))
    assert st == g.GD_OK and order == [0, 2, 1]


def test_round_robin_fifo_and_fairness():
    rng = np.random.Generator(np.random.PCG64(11))
    for _ in range(200):
        tenants = [int(x) for x in rng.integers(0, 6, int(rng.integers(1, 60)))]
        st, order = g.gd_schedule_round_robin(_items(tenants))
        assert st == g.GD_OK and sorted(order) == list(range(len(tenants)))
        # FIFO within a tenant
        for t in set(tenants):
            seq = [i for i in order if tenants[i] == t]
            assert seq == sorted(seq)
        # round-robin: in every prefix no tenant is more than one launch ahead
        # of another tenant that still has work queued
        total = {t: tenants.count(t) for t in set(tenants)}
        issued = {t: 0 for t in total}
        for i in order:
            issued[tenants[i]] += 1
            for x in total:
                for y in total:
                    if issued[y] < total[y]:
                        assert issued[x] <= issued[y] + 1


def test_launcher_validates_all_before_issuing():
    a = virtual()
    p = a.partition_alloc(1 << 20)
    items = [g.work(p.id, g.GD_KIND_COPY, "mask", ptr=(p.base, p.base), u64=(0,)),
             g.work(p.id, g.GD_KIND_COPY, "mask", ptr=(p.base + 8, p.base), u64=(64,))]
    with pytest.raises(g.GuardianError) as e:
        a.launcher_run(items, [None])
    assert e.value.status == g.GD_ERR_ALIGN
    assert a.stats(p.id)["launches"] == 0


@pytest.mark.parametrize("policy", ["round_robin", "no_tensor_random", "memory_lane"])
def test_launcher_policies_validate_before_issuing(policy):
    """Every issue policy validates all items first (nothing issued, nothing
    counted on a bad item); an unknown policy is refused before anything."""
    a = virtual()
    p = a.partition_alloc(1 << 20)
    good = g.work(p.id, g.GD_KIND_COPY, "mask", ptr=(p.base, p.base), u64=(0,))
    bad = g.work(p.id, g.GD_KIND_GEMM, "check", ptr=(p.base, p.base, p.base), u64=(64, 64, 64), u32=(64, 64, 63))
    with pytest.raises(g.GuardianError) as e:
        a.launcher_run([good, bad], [None, None], policy=policy)
    assert e.value.status == g.GD_ERR_UNSUPPORTED
    assert a.stats(p.id)["launches"] == 0
    with pytest.raises(g.GuardianError) as e:
        a.launcher_run([good], [None], policy=7)
    assert e.value.status == g.GD_ERR_INVALID_ARG
    a.launcher_run([good], [None], policy=policy)        # n = 0 work: valid, nothing launched


def test_native_when_solo_setter():
    a = virtual()
    a.set_native_when_solo(True)
    a.set_native_when_solo(False)


def test_exact_partitions_tail_returns_to_pool():
    """gd_partition_alloc_exact: a 12 KiB request takes a
    16 KiB block and gives the 4 KiB tail back, which a later 4 KiB request
    receives; freeing coalesces everything back to one block."""
    a = virtual(1 << 20)
    x = a.partition_alloc_exact(12 << 10)
    assert x.size == 12 << 10 and not x.pow2 and x.base == DEV_BASE
    y = a.partition_alloc(4 << 10)
    assert y.base == DEV_BASE + (12 << 10)              # the returned tail
    with pytest.raises(g.GuardianError) as e:
        a.copy(x.id, "mask", x.base, x.base + 16, 64)
    assert e.value.status == g.GD_ERR_NOT_POW2
    with pytest.raises(g.GuardianError) as e:           # modulo / check accepted (no device)
        a.copy(x.id, "modulo", x.base, x.base + 16, 64)
    assert e.value.status == g.GD_ERR_UNSUPPORTED
    a.partition_free(x.id)
    a.partition_free(y.id)
    z = a.partition_alloc(1 << 20)                      # fully coalesced again
    assert z.base == DEV_BASE


@pytest.mark.parametrize("seed", [3, 4])
def test_mixed_exact_and_pow2_fuzz_against_bitmap(seed):
    """Exact and power-of-two partitions mixed: disjoint, inside the arena,
    pow2 ones size-aligned, exact ones 4 KiB-aligned and sized; all space
    comes back after freeing everything."""
    size = 1 << 24
    a = virtual(size)
    ref = BitmapArena(DEV_BASE, size)
    rng = np.random.Generator(np.random.PCG64(seed))
    live = {}
    for _ in range(800):
        if live and (rng.random() < 0.45 or len(live) >= 60):
            pid = int(rng.choice(list(live)))
            a.partition_free(pid)
            b, s = live.pop(pid)
            lo = (b - DEV_BASE) // 4096
            ref.used[lo:lo + s // 4096] = False
        else:
            req = int(2 ** rng.uniform(0, 22))
            exact = rng.random() < 0.5
            try:
                p = a.partition_alloc_exact(req) if exact else a.partition_alloc(req)
            except g.GuardianError as e:
                assert e.status == g.GD_ERR_DEVICE_OOM
                continue
            if exact:
                assert p.size == max(4096, -(-req // 4096) * 4096) and p.base % 4096 == 0
            else:
                assert p.size == partition_size(req) and p.base % p.size == 0
            lo = (p.base - DEV_BASE) // 4096
            assert not ref.used[lo:lo + p.size // 4096].any() and p.base + p.size <= DEV_BASE + size
            ref.used[lo:lo + p.size // 4096] = True
            live[p.id] = (p.base, p.size)
    for pid in list(live):
        a.partition_free(pid)
    assert a.partition_alloc(size).base == DEV_BASE
