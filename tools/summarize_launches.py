"""Summarise an ncu launch list (gpu__time_duration.sum per launch) into
per-kernel counts, mean duration and share of the total: the kernel SHARE of
the step is what must agree with bench.py's live roofline numbers."""
import collections
import csv
import json
import re
import sys


def main(path, out):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ki, vi, mi, gi = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Name"), hdr.index("Grid Size")
    agg = collections.OrderedDict()
    for r in rows[1:]:
        if r[mi] != "gpu__time_duration.sum":
            continue
        name = re.sub(r"<.*>", "", re.sub(r"^.*::", "", r[ki].split("(")[0]))
        m = re.search(r"<(\d)>", r[ki])
        if "<" in r[ki] and m:
            name += f"<{ {'0': 'none', '1': 'mask', '2': 'check', '3': 'modulo', '4': 'maskcount', '5': 'clamp', '6': 'mask_big'}[m.group(1)] }>"
        d = agg.setdefault(name, {"launches": 0, "total_ns": 0.0, "grid": r[gi]})
        d["launches"] += 1
        d["total_ns"] += float(r[vi].replace(",", ""))
    tot = sum(d["total_ns"] for d in agg.values())
    for d in agg.values():
        d["mean_us"] = round(d["total_ns"] / d["launches"] / 1e3, 2)
        d["share"] = round(d["total_ns"] / tot, 4)
    # share of each kernel within the timed bench step (C2, mask: one copy and
    # one saxpy per tenant): what bench.py's roofline.share_of_step measures live
    # (mask on the bench's 16 GiB partitions launches the internal mask_big
    # instantiation, fence_desc.h kMaskBig)
    step = [k for k in ("k_copy<mask>", "k_saxpy<mask>") if k in agg] or \
        [k for k in ("k_copy<mask_big>", "k_saxpy<mask_big>") if k in agg]
    step_tot = sum(agg[k]["mean_us"] for k in step)
    step_share = {k: round(agg[k]["mean_us"] / step_tot, 4) for k in step} if step_tot else {}
    json.dump({"source": path, "note": "ncu --metrics gpu__time_duration.sum --clock-control none; cold-cache, "
               "serialised launches: compare shares, not absolutes", "step_share_c2_mask": step_share,
               "kernels": agg}, open(out, "w"), indent=1)
    print("share within the C2 mask step:", step_share)
    for k, d in agg.items():
        print(f"{k:24s} n={d['launches']:5d} mean={d['mean_us']:10.2f} us share={d['share']:.3f} grid={d['grid']}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
