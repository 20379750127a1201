#!/bin/bash
# GEMM raster-group probe: time (interleaved with cuBLAS) and ncu DRAM bytes per group size.
cd "$(dirname "$0")/.."
for G in 4 8 16 32; do
  echo "== group $G"
  GD_GEMM_GROUP=$G timeout 300 python tools/kernel_bench.py --reps 6 --only gemm 2>&1 | grep -E "gemm|torch"
  GD_GEMM_GROUP=$G timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed -k regex:k_gemm -c 1 python tools/prof_kernel.py --kind gemm --mode mask --reps 1 2>&1 | grep -E "duration|dram__bytes|tensor"
done
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed -c 3 python -c "
import torch; a=torch.randn(8192,8192,dtype=torch.bfloat16,device='cuda'); b=torch.randn(8192,8192,dtype=torch.bfloat16,device='cuda')
for _ in range(3): c=torch.matmul(a,b.t())
torch.cuda.synchronize()" 2>&1 | grep -E "nvjet|cutlass|sm100|gemm|duration|dram__bytes|tensor" | head -20
