#!/bin/bash
# Final evidence of a round in one GPU call: every GPU test, smoke, bench.py x 3, the ncu launch
# list of the bench, ncu --set full of the stencil (hoisted and per access).  Output in gpurun_out/.
cd "$(dirname "$0")/.."
NCU=1 bash tools/gpu_round.sh > gpurun_out/fin_round.txt 2>&1
for i in 2 3; do timeout 900 python bench.py > gpurun_out/bench_$i.json 2> gpurun_out/bench_$i.err; done
bash tools/ncu_full.sh "stencil:mask stencil:check" > gpurun_out/fin_ncu_h.txt 2>&1
for m in check modulo; do
  GD_CHECK_PER_ACCESS=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_stencil_pa -s 1 -c 1 \
    -o gpurun_out/prof_stencilpa_$m -f python tools/prof_kernel.py --kind stencil --mode $m --reps 2 > gpurun_out/ncu_stencilpa_$m.log 2>&1
done
echo FINAL_DONE
