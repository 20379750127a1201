#!/bin/bash
# A/B: row-gather clamp code generation per slot width (cs2 / ns2 / rd2 / all2
# vs now10); placement probe of the L2-resident per-access gather (KB_SLOTS).
cd "$(dirname "$0")/.."
O=gpurun_out/r02it11; mkdir -p $O
M=none,clamp,clamp+pa,modulo+pa,check+pa,maskcount+pa
for v in now10 cs2 ns2 rd2 all2; do
  GD_LIB=tools/variants/lib_$v.so timeout 600 python tools/kernel_bench.py --reps 12 --only gatherrows --modes $M > $O/kbg_$v.json 2> $O/kbg_$v.txt
done
for sl in 2 8; do
  KB_SLOTS=$sl GD_LIB=tools/variants/lib_now10.so timeout 600 python tools/kernel_bench.py --reps 12 --only l2 --modes none,mask,check,check+pa,modulo+pa,maskcount+pa > $O/kbl2_s$sl.json 2> $O/kbl2_s$sl.txt
done
for v in now10 cs2 ns2 rd2 all2; do echo "== $v"; cat $O/kbg_$v.txt; done; for sl in 2 8; do echo "== slots $sl"; grep -i "gather\|stencil 2048" $O/kbl2_s$sl.txt; done
