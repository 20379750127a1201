#!/bin/bash
cd "$(dirname "$0")/.."
O=gpurun_out/r02p4; mkdir -p $O
prof() {
  local name=$1 kre=$2; shift 2
  timeout 600 ncu --set full --clock-control none --import-source on -k "regex:${kre}" -s 1 -c 1 \
      -o $O/$name -f python tools/prof_kernel.py --reps 2 "$@" > $O/$name.log 2>&1
}
prof gr64_clamp k_gatherR --kind gatherrows --D 64 --mode clamp
prof gr64_check k_gatherR --kind gatherrows --D 64 --mode check
prof gr32_clamp k_gatherR --kind gatherrows --D 32 --mode clamp
prof gr32_check k_gatherR --kind gatherrows --D 32 --mode check
prof st_l2_check_pa k_stencil_pa --kind stencil --mode check --l2 --pa
prof st_l2_none k_stencil --kind stencil --mode none --l2
M=none,mask,check,modulo,maskcount,clamp,check+pa,modulo+pa,maskcount+pa,clamp+pa
timeout 900 python tools/kernel_bench.py --reps 10 --only stencil,l2 --modes $M > $O/kb.json 2> $O/kb.txt
cat $O/kb.txt
