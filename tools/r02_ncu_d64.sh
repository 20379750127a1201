#!/bin/bash
# ncu --set full of the D = 64 row gather: none vs clamp vs mask (hoisted)
cd "$(dirname "$0")/.."
O=gpurun_out/r02ncud64; mkdir -p $O
for m in none clamp mask; do
  timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:k_gatherR" -s 1 -c 1 \
      -o $O/prof_$m -f python tools/prof_kernel.py --reps 2 --kind gatherrows --D 64 --mode $m > $O/prof_$m.log 2>&1
  ncu -i $O/prof_$m.ncu-rep --page raw --csv > $O/raw_$m.csv 2>/dev/null
  ncu -i $O/prof_$m.ncu-rep --page source --csv > $O/src_$m.csv 2>/dev/null
done
rm -f $O/*.ncu-rep
ls -la $O
