#!/bin/bash
# Tuning-knob probe: the 2-SM GEMM's TMA L2 eviction hints (GD_GEMM_L2HINT:
# 0 normal, 1 A evict_last + B evict_first, 2 A evict_last, 3 half of A
# evict_last), each timed with kernel_bench (interleaved with cuBLAS) and
# with ncu DRAM bytes per launch.
cd "$(dirname "$0")/.."
for H in ${HINTS:-0 1 2 3}; do
  echo "== GD_GEMM_L2HINT=$H"
  GD_GEMM_L2HINT=$H timeout 300 python tools/kernel_bench.py --reps 6 --only gemm 2>&1 | grep -E "^gemm|torch"
  GD_GEMM_L2HINT=$H timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed -k regex:k_gemm -c 1 python tools/prof_kernel.py --kind gemm --mode mask --reps 1 2>&1 | grep -E "duration|dram__bytes|tensor"
done
