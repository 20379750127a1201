#!/bin/bash
# ncu --set full captures of the fenced kernels (one GPU, one kernel each).
# usage: tools/ncu_full.sh "saxpy:mask copy:mask gather:mask gemm:mask"
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for kv in ${1:-saxpy:mask}; do
  kind=${kv%%:*}; mode=${kv##*:}
  kre="k_${kind}"; extra=""
  if [ "$kind" = gatherrows ]; then kre="k_gatherR"; extra="--D 32"; fi
  if [ "$kind" = stencil_tma ]; then kre="k_stencil_tma"; fi
  timeout 600 ncu --set full --clock-control none --import-source on -k "regex:${kre}" -s 1 -c 1 \
      -o gpurun_out/prof_${kind}_${mode} -f python tools/prof_kernel.py --kind $kind --mode $mode --reps 2 $extra \
      > gpurun_out/ncu_${kind}_${mode}.log 2>&1
  echo "ncu $kind $mode rc=$?" >> gpurun_out/ncu_${kind}_${mode}.log
  tail -2 gpurun_out/ncu_${kind}_${mode}.log
done
