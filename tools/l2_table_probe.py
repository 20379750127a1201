"""Why does bench.py's L2-resident per-access gather cost more than
tools/kernel_bench.py's?  Runs bench.Workload's l2_table (per access) in a
fresh process, then after the bench's HBM per-access kernel table, then again.
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402


def show(tag, t):
    print(tag, json.dumps({k: {m: round(100 * (v["ms"] / row["none"]["ms"] - 1), 2) for m, v in row.items()}
                           for k, row in t.items() if "gather" in k or "stencil_2048" in k}), flush=True)


def main():
    import torch
    torch.cuda.set_device(0)
    w = bench.Workload(0)
    w.c5_setup()
    w.rows_setup()
    show("l2 pa, fresh:", w.l2_table(reps=6, per_access=True))
    show("l2, fresh:", w.l2_table(reps=6))
    w.kernel_table(reps=6, per_access=True)
    show("l2 pa, after the HBM per-access table:", w.l2_table(reps=6, per_access=True))
    w.kernel_table(reps=6)
    show("l2 pa, after both HBM tables:", w.l2_table(reps=6, per_access=True))


if __name__ == "__main__":
    main()
