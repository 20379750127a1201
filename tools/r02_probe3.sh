#!/bin/bash
# Round-2 probe 3: per-stage times of the bucketed scatter; re-measure stencil + gather rows.
cd "$(dirname "$0")/.."
O=gpurun_out/r02p3; mkdir -p $O
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed,lts__t_sector_hit_rate.pct,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none -k "regex:k_scatter" --csv --log-file $O/scatter_stages.csv python tools/prof_kernel.py --kind scatter --mode mask --reps 2 > $O/scatter_stages.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:k_scatter_apply" -s 1 -c 1 -o $O/scatter_apply -f python tools/prof_kernel.py --kind scatter --mode mask --reps 2 > $O/scatter_apply.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:k_scatter_part" -s 2 -c 2 -o $O/scatter_part -f python tools/prof_kernel.py --kind scatter --mode mask --reps 2 > $O/scatter_part.log 2>&1
M=none,mask,check,modulo,maskcount,clamp,check+pa,modulo+pa,maskcount+pa,clamp+pa
timeout 900 python tools/kernel_bench.py --reps 10 --only stencil,gatherrows,gather --modes $M > $O/kb.json 2> $O/kb.txt
cat $O/kb.txt; python - <<'PY'
import csv
rows=list(csv.reader(open("gpurun_out/r02p3/scatter_stages.csv")))
h=None
for r in rows:
    if "Kernel Name" in r: h=r; continue
    if h and len(r)==len(h): print(r[h.index("Kernel Name")][:40], r[h.index("Metric Name")], r[h.index("Metric Value")])
PY
