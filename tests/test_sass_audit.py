"""Static audit of the sm_100a machine code in libguardian.so (CPU only:
cuobjdump disassembles without a GPU).

* No kernel touches local memory (LDL/STL): there is nothing unfenced on a
  stack (reading A13; PAPER.md:127 protects local memory).
* No indirect branches (BRX/JMX): nothing for a `brx.idx` attack to use
  (SURVEY M14).
* The GEMM really runs on the 5th-generation tensor cores with TMA
  (UTC*MMA, UTMALDG) and not on the legacy HMMA path.
* Every fenced variant carries extra fence logic over its unfenced twin:
  mask / modulo variants execute more LOP3 / IMAD.HI work than NONE.
"""
import re
import subprocess

import pytest

from paper_2401_09290_b200 import guardian as g


@pytest.fixture(scope="module")
def sass():
    txt = subprocess.run(["cuobjdump", "-sass", g.LIB_PATH], capture_output=True, text=True).stdout
    funcs = re.split(r"\n\s*Function : ", txt)[1:]
    names = [f.split("\n", 1)[0].strip() for f in funcs]
    dm = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True).stdout.split("\n")
    out = {}
    for body, name in zip(funcs, dm):
        ins = re.findall(r"/\*[0-9a-f]{4}\*/\s+(?:@!?U?P\w+\s+)?([A-Z0-9_.]+)", body)
        short = re.sub(r"\(.*", "", name.replace("gd::(anonymous namespace)::", "").replace("void ", ""))
        out[short] = ins
    assert len(out) >= 20
    return out


def count(ins, pat):
    return sum(1 for i in ins if re.match(pat, i))


def test_no_local_memory_no_indirect_branches(sass):
    for name, ins in sass.items():
        assert count(ins, r"(LDL|STL)\b") == 0, name
        assert count(ins, r"(BRX|JMX)\b") == 0, name


def test_gemm_uses_tcgen05_and_tma(sass):
    for k in ("k_gemm", "k_gemm2"):
        ins = sass[k]
        assert count(ins, r"UTC\w*MMA") >= 1, k
        assert count(ins, r"UTMALDG") >= 2, k
        assert count(ins, r"HMMA") == 0, k
    assert any(i.startswith("UTMALDG.2D.2CTA") for i in sass["k_gemm2"])


def test_stencil_v2_is_tma_staged(sass):
    """K5 v2 moves its tiles with TMA (load and store) and has no per-access
    global load or store besides the <= 3 tail columns."""
    ins = sass["k_stencil_tma"]
    assert count(ins, r"UTMALDG") >= 1 and count(ins, r"UTMASTG") >= 1
    assert count(ins, r"LDG") == 0


@pytest.mark.parametrize("kernel", ["k_copy", "k_saxpy", "k_gather1", "k_gatherE", "k_scatter", "k_stencil"])
def test_fenced_variants_carry_fence_logic(sass, kernel):
    def key(m):            # k_x<m> or k_x<m, ...> (first instantiation)
        keys = sorted(k for k in sass if k == f"{kernel}<{m}>" or k.startswith(f"{kernel}<{m},"))
        assert keys, (kernel, m)
        return keys[0]
    none, mask, modulo = sass[key(0)], sass[key(1)], sass[key(3)]
    assert count(mask, r"LOP3") > count(none, r"LOP3"), kernel
    assert count(modulo, r"IMAD\.(WIDE\.)?HI|IMAD\.HI") + count(modulo, r"IMAD\.WIDE") > \
        count(none, r"IMAD\.(WIDE\.)?HI|IMAD\.HI") + count(none, r"IMAD\.WIDE"), kernel
    # same memory instructions in the fenced variant as in the twin (the fence
    # changes addresses, not the access pattern); the mask stencil has one more
    # copy of its full-strip path, specialised for >= 4 GiB partitions
    # (Fence::addr_big): 2 + ROWS vector loads, ROWS halo loads, ROWS stores
    extra = 0
    if kernel == "k_stencil":
        rows = int(re.search(r"<1, (\d+)>", key(1)).group(1))
        extra = 2 + 3 * rows
    assert count(mask, r"(LDG|STG|ATOM|RED)") == count(none, r"(LDG|STG|ATOM|RED)") + extra, kernel
