#!/bin/bash
# ncu of the scatter-add v2 partition passes, none vs mask vs check per
# access, 0 % out-of-partition indices; kernel bench of the scatter.
cd "$(dirname "$0")/.."
O=gpurun_out/r02ncu3; mkdir -p $O
run() {  # name, args...
  local n=$1; shift
  timeout 600 ncu --set full --clock-control none --import-source on -k "regex:k_scatter_part" -s 2 -c 2 \
      -o $O/$n -f python tools/prof_kernel.py --kind scatter --reps 3 --oob 0 "$@" > $O/$n.log 2>&1
  echo "$n rc=$?" >> $O/$n.log; tail -1 $O/$n.log
}
run sc_none --mode none
run sc_mask --mode mask
run sc_check_pa --mode check --pa
M=none,mask,check,modulo,maskcount,clamp,check+pa,modulo+pa,maskcount+pa,clamp+pa
timeout 600 python tools/kernel_bench.py --reps 12 --only scatter --modes $M > $O/kb.json 2> $O/kb.txt
cat $O/kb.txt
