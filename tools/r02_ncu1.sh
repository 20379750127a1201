#!/bin/bash
# ncu --set full of the stencil: HBM per access (none / check / clamp /
# maskcount) and L2-resident hoisted (none / mask / check); kernel bench of
# the current build twice (run-to-run spread).
cd "$(dirname "$0")/.."
O=gpurun_out/r02ncu1; mkdir -p $O
run() {  # name, args...
  local n=$1; shift
  timeout 600 ncu --set full --clock-control none --import-source on -k "regex:k_stencil" -s 1 -c 1 \
      -o $O/$n -f python tools/prof_kernel.py --kind stencil --reps 2 "$@" > $O/$n.log 2>&1
  echo "$n rc=$?" >> $O/$n.log; tail -1 $O/$n.log
}
run hbm_none --mode none
run hbm_check_pa --mode check --pa
run hbm_clamp_pa --mode clamp --pa
run hbm_maskcount_pa --mode maskcount --pa
run l2_none --mode none --l2
run l2_mask --mode mask --l2
run l2_check --mode check --l2
M=none,mask,check,maskcount,check+pa,modulo+pa,maskcount+pa,clamp+pa
for r in 1 2; do
  timeout 600 python tools/kernel_bench.py --reps 12 --only stencil,gatherrows,l2 --modes $M > $O/kb_now2_$r.json 2> $O/kb_now2_$r.txt
done
for r in 1 2; do echo "== run $r"; cat $O/kb_now2_$r.txt; done
