#!/bin/bash
# Round-2 probe 1 (one GPU call): scatter limiter probe, ncu --set full of the
# scatter / D=1 gather / per-access stencil and row gather, per-access baseline.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/r02p1
O=gpurun_out/r02p1
timeout 300 python tools/scatter_probe.py > $O/scatter_probe.json 2> $O/scatter_probe.txt
prof() {  # name kernel-regex env args...
  local name=$1 kre=$2; shift 2
  timeout 600 env "$@" ncu --set full --clock-control none --import-source on -k "regex:${kre}" -s 1 -c 1 \
      -o $O/$name -f python tools/prof_kernel.py --reps 2 ${PK_ARGS} > $O/$name.log 2>&1
  echo "rc=$?" >> $O/$name.log
}
PK_ARGS="--kind scatter --mode mask" prof scatter_mask k_scatter GD_X=0
PK_ARGS="--kind gather --mode mask" prof gather_mask k_gather1 GD_X=0
PK_ARGS="--kind stencil --mode none" prof stencil_none k_stencil GD_X=0
PK_ARGS="--kind stencil --mode check" prof stencil_pa_check k_stencil_pa GD_CHECK_PER_ACCESS=1
PK_ARGS="--kind stencil --mode mask" prof stencil_mask k_stencil GD_X=0
PK_ARGS="--kind gatherrows --mode none" prof gatherR_none k_gatherR GD_X=0
PK_ARGS="--kind gatherrows --mode modulo" prof gatherR_pa_modulo k_gatherR GD_CHECK_PER_ACCESS=1
M=none,mask,check,modulo,maskcount,clamp
GD_CHECK_PER_ACCESS=1 timeout 900 python tools/kernel_bench.py --reps 8 --only stencil,gatherrows,l2 --modes $M > $O/kb_pa.json 2> $O/kb_pa.txt
timeout 900 python tools/kernel_bench.py --reps 8 --only stencil,l2 --modes $M > $O/kb_hoist.json 2> $O/kb_hoist.txt
cat $O/scatter_probe.txt; cat $O/kb_pa.txt $O/kb_hoist.txt; tail -n 2 $O/*.log
