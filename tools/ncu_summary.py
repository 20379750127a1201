"""Summarise ncu --set full reports into profiles/<tag>.json (+ print).

  python tools/ncu_summary.py gpurun_out/prof_saxpy_mask.ncu-rep ... --out profiles/r01_ncu.json
Also updates profiles/ncu_traffic.json: {"k_<kind><mode_id>": dram bytes per launch}
(bench.py's roofline.traffic).
"""
import csv
import io
import json
import os
import re
import subprocess
import sys

METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram__cycles_active.avg.pct_of_peak_sustained_elapsed",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram__bytes.sum.per_second",
    "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread", "launch__grid_size",
    "launch__block_size", "launch__occupancy_limit_registers", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "lts__t_sector_hit_rate.pct", "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum",
    "lts__t_sectors_srcunit_tex_op_read.sum", "smsp__inst_executed.sum",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_op_gmma_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_uniform.avg.pct_of_peak_sustained_active",
    "smsp__average_warp_latency_issue_stalled_long_scoreboard.pct",
    "launch__shared_mem_per_block_dynamic", "sm__cycles_elapsed.avg.per_second",
]


def read(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, u = rows[0], rows[1]
    res = []
    for v in rows[2:]:
        d = {"kernel": v[h.index("Kernel Name")]}
        for i, n in enumerate(h):
            if n in METRICS or re.search(r"tensor.*pct_of_peak_sustained_(active|elapsed)$", n) and "max" not in n \
                    and "min" not in n and "sum" not in n:
                try:
                    val = float(v[i].replace(",", ""))
                except ValueError:
                    continue
                if val == 0 and "tensor" in n:
                    continue
                d[n] = {"value": val, "unit": u[i]}
        res.append(d)
    return res


def to_bytes(m):
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
    return m["value"] * scale.get(m["unit"], 1)


def main():
    args = sys.argv[1:]
    out = args[args.index("--out") + 1] if "--out" in args else None
    reps = [a for a in args if a.endswith(".ncu-rep")]
    summary = {}
    tpath = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "ncu_traffic.json")
    if "--traffic" in args:                            # e.g. on the GPU box: a copy under gpurun_out/
        tpath = args[args.index("--traffic") + 1]
    traffic = json.load(open(tpath)) if os.path.exists(tpath) else {}
    for rep in reps:
        for d in read(rep):
            name = d["kernel"]
            tag = os.path.basename(rep).replace(".ncu-rep", "")
            summary[tag] = d
            print(f"== {tag}: {name}")
            for k, m in d.items():
                if k != "kernel":
                    print(f"   {k:72s} {m['value']:>16.4f} {m['unit']}")
            if "dram__bytes_read.sum" in d:
                rd, wr = to_bytes(d["dram__bytes_read.sum"]), to_bytes(d["dram__bytes_write.sum"])
                mm = re.search(r"(k_[A-Za-z0-9]+)<([\d, ]+)>", name)
                key = (f"{mm.group(1)}<{mm.group(2).replace(' ', '')}>" if mm
                       else re.sub(r"^.*::", "", re.sub(r"\(.*", "", name)))
                traffic[key] = rd + wr
                # ncu's DRAM throughput, % of its theoretical peak (B200: 2048 B per
                # DRAM cycle x 3.996 GHz = 8.18 TB/s); this ncu reports it as
                # gpu__dram_throughput (dram__throughput reads "-")
                for pm in ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
                           "dram__throughput.avg.pct_of_peak_sustained_elapsed"):
                    if pm in d:
                        traffic[key + ":dram_pct"] = d[pm]["value"]
                        break
                traffic["_source"] = f"ncu --set full, {os.path.basename(rep)}"
                print(f"   traffic (dram read+write) = {rd + wr:.4e} B")
    if out:
        json.dump(summary, open(out, "w"), indent=1)
    json.dump(traffic, open(tpath, "w"), indent=1)


if __name__ == "__main__":
    main()
