"""Register / local-memory report of the fenced kernels against their unfenced
twins, from the ptxas -v logs of the build (the paper's
Figure 9 / PAPER.md:369-371 reports extra registers of sandboxed kernels:
71 % +0, 13 % +1, 7 % +2 at -O3).

  python tools/register_report.py [--out profiles/r01_registers.json]
"""
import glob
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BUILD = os.path.join(ROOT, "paper_2401_09290_b200", "build")
MODES = {"0": "none", "1": "mask", "2": "check", "3": "modulo", "4": "maskcount", "5": "clamp",
         "6": "mask_big"}  # 6: internal, mask on a >= 4 GiB partition (fence_desc.h kMaskBig)


def demangle(names):
    out = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True).stdout.split("\n")
    return dict(zip(names, out))


def ctas_by_regs(regs, threads=256):
    """CTAs of `threads` per SM the register file allows (64 K registers per
    SM, allocated per warp in units of 256 registers)."""
    per_warp = -(-regs * 32 // 256) * 256
    return (65536 // per_warp) // (threads // 32)


def main():
    rows = {}
    for log in sorted(glob.glob(os.path.join(BUILD, "ptxas_*.log"))):
        txt = open(log).read()
        for m in re.finditer(r"Function properties for (\S+)\n\s+(\d+) bytes stack frame, (\d+) bytes spill stores, "
                             r"(\d+) bytes spill loads\nptxas info\s+: Used (\d+) registers", txt):
            rows[m.group(1)] = {"stack": int(m.group(2)), "spill_st": int(m.group(3)), "spill_ld": int(m.group(4)),
                                "regs": int(m.group(5))}
    dm = demangle(list(rows))
    table = {}
    for mangled, r in rows.items():
        name = dm[mangled]
        km = re.search(r"(k_[A-Za-z0-9_]+)<(\d)((?:, ?[\w]+)*)>", name)
        if not km:
            continue
        # one row per instantiation (the other template arguments kept), so
        # every fenced variant is compared with the twin of the same shape
        rest = km.group(3).replace(" ", "")
        kernel, mode = km.group(1) + (f"<M{rest}>" if rest else ""), MODES.get(km.group(2), km.group(2))
        table.setdefault(kernel, {})[mode] = r
    report = {"source": "ptxas -v of the sm_100a build (paper_2401_09290_b200/build/ptxas_*.log)", "kernels": {}}
    deltas = []
    for k, modes in sorted(table.items()):
        if "none" not in modes:
            continue
        base = modes["none"]["regs"]
        # every kernel here runs 256-thread CTAs; the occupancy that matters
        # is the register-limited CTA count (each kernel's __launch_bounds__
        # caps it anyway), so report it beside the raw register delta
        occ0 = ctas_by_regs(base)
        report["kernels"][k] = {m: dict(v, delta_regs=v["regs"] - base, ctas_per_sm_by_regs=ctas_by_regs(v["regs"]),
                                        occupancy_change=ctas_by_regs(v["regs"]) - occ0)
                                for m, v in modes.items()}
        for m, v in modes.items():
            if m != "none":
                deltas.append(v["regs"] - base)
                assert v["stack"] == 0 and v["spill_st"] == 0, (k, m, v)     # reading A13: no local memory
    hist = {}
    for d in deltas:
        hist[str(d)] = hist.get(str(d), 0) + 1
    report["delta_histogram"] = dict(sorted(hist.items(), key=lambda kv: int(kv[0])))
    report["all_zero_local_memory"] = all(v["stack"] == 0 for m in table.values() for v in m.values())
    report["fenced_variants_with_lower_occupancy"] = sorted(
        f"{k}/{m}" for k, ms in report["kernels"].items() for m, v in ms.items() if v["occupancy_change"] < 0)
    for k, modes in report["kernels"].items():
        print(f"{k:12s} " + "  ".join(f"{m}:{v['regs']}({v['delta_regs']:+d})" for m, v in modes.items()))
    print("delta histogram (fenced - unfenced registers):", report["delta_histogram"])
    print("fenced variants with fewer register-limited CTAs per SM than their twin:",
          report["fenced_variants_with_lower_occupancy"])
    if "--out" in sys.argv:
        json.dump(report, open(sys.argv[sys.argv.index("--out") + 1], "w"), indent=1)


if __name__ == "__main__":
    main()
