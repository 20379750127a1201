#!/bin/bash
# ncu of the L2-resident stencil with --cache-control none (the replays see a
# warm L2, as the graph-replayed bench does): none / mask / check hoisted /
# check per access; and the D = 32 row gather per access (none / check /
# modulo / clamp) at HBM size.
cd "$(dirname "$0")/.."
O=gpurun_out/r02ncu2; mkdir -p $O
run() {  # name, kernel regex, args...
  local n=$1 k=$2; shift 2
  timeout 600 ncu --set full --cache-control none --clock-control none --import-source on -k "regex:$k" -s 2 -c 1 \
      -o $O/$n -f python tools/prof_kernel.py --reps 4 "$@" > $O/$n.log 2>&1
  echo "$n rc=$?" >> $O/$n.log; tail -1 $O/$n.log
}
run l2_none k_stencil --kind stencil --mode none --l2
run l2_mask k_stencil --kind stencil --mode mask --l2
run l2_check k_stencil --kind stencil --mode check --l2
run l2_check_pa k_stencil --kind stencil --mode check --l2 --pa
run g32_none k_gatherR --kind gatherrows --D 32 --mode none
run g32_check_pa k_gatherR --kind gatherrows --D 32 --mode check --pa
run g32_modulo_pa k_gatherR --kind gatherrows --D 32 --mode modulo --pa
run g32_clamp_pa k_gatherR --kind gatherrows --D 32 --mode clamp --pa
