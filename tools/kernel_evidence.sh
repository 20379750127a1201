#!/bin/bash
# Kernel-level evidence in one GPU call: every kernel in all six modes
# (hoisted default), the hoisted and per-access (GD_CHECK_PER_ACCESS=1) runs
# incl. the L2-resident sizes.  Output in gpurun_out/kb_*.json.
cd "$(dirname "$0")/.."
M=none,mask,check,modulo,maskcount,clamp
K=copy,saxpy,gather,scatter,stencil,stencil_tma,gatherrows,l2
timeout 1200 python tools/kernel_bench.py --modes $M > gpurun_out/kb_6modes.json 2> gpurun_out/kb_6modes.err
timeout 900 python tools/kernel_bench.py --only $K --modes $M > gpurun_out/kb_hoist.json 2> gpurun_out/kb_hoist.err
GD_CHECK_PER_ACCESS=1 timeout 900 python tools/kernel_bench.py --only $K --modes $M > gpurun_out/kb_peraccess.json 2> gpurun_out/kb_pa.err
