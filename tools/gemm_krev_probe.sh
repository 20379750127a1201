#!/bin/bash
# GEMM K-direction alternation (GD_GEMM_KREV) x raster group (GD_GEMM_GROUP):
# sustained TFLOP/s interleaved with cuBLAS, and ncu DRAM bytes per launch.
cd "$(dirname "$0")/.."
for KR in 0 1; do for G in ${GRPS:-8 16}; do
  echo "== KREV=$KR GROUP=$G"
  GD_GEMM_KREV=$KR GD_GEMM_GROUP=$G timeout 300 python tools/kernel_bench.py --reps 6 --modes none,mask --only gemm 2>&1 | grep -E "^gemm|torch"
  GD_GEMM_KREV=$KR GD_GEMM_GROUP=$G timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed -k regex:k_gemm -c 1 python tools/prof_kernel.py --kind gemm --mode mask --reps 1 2>&1 | grep -E "duration|dram__bytes|tensor"
done; done
