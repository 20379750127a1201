#!/bin/bash
# ncu --set full of the random-access kernels at 0 % out-of-partition indices
# (the unfenced twin on planted indices would leave prof_kernel's one-partition
# arena): D = 1 gather, scatter-add v2 pass A3 and apply, none / mask / check.
cd "$(dirname "$0")/.."
O=gpurun_out/r02rand; mkdir -p $O
cap() {  # name, kernel regex, skip, prof_kernel args...
  local n=$1 k=$2 sk=$3; shift 3
  timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:$k" -s $sk -c 1 \
      -o $O/prof_$n -f python tools/prof_kernel.py --reps 2 --oob 0 "$@" > $O/prof_$n.log 2>&1
  echo "$n rc=$?" >> $O/prof_$n.log; tail -1 $O/prof_$n.log
}
for m in none mask check; do
  cap gather_$m "k_gather1<" 1 --kind gather --mode $m
  cap scatterA3_$m "k_scatter_part<.int.[0-9], .int.1>" 1 --kind scatter --mode $m
  cap scatterB_$m "k_scatter_apply" 1 --kind scatter --mode $m
done
python tools/ncu_summary.py $O/prof_*.ncu-rep --out $O/ncu_rand.json --traffic $O/ncu_traffic_rand.json > $O/ncu_rand.txt 2>&1
rm -f $O/prof_*.ncu-rep
du -sh $O
