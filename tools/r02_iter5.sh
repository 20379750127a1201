#!/bin/bash
# A/B: check-mode stencil loads at the mask-fenced address + zero fix-up (now3
# vs cm0), row-gather clamp / live-slot variants (cs, cs_nosw, live).
cd "$(dirname "$0")/.."
O=gpurun_out/r02it5; mkdir -p $O
timeout 900 python -m pytest -q -p no:cacheprovider -m gpu -x tests/test_gpu_kernels.py tests/test_gpu_count_modes.py tests/test_gpu_peraccess.py tests/test_gpu_fullscale.py -k "stencil" > $O/pytest.log 2>&1
echo "rc=$?" >> $O/pytest.log
M=none,mask,check,maskcount,check+pa,modulo+pa,maskcount+pa,clamp+pa
for v in now3 cm0; do
  GD_LIB=tools/variants/lib_$v.so timeout 600 python tools/kernel_bench.py --reps 12 --only stencil,l2 --modes $M > $O/kb_$v.json 2> $O/kb_$v.txt
done
for v in now3 cs cs_nosw live; do
  GD_LIB=tools/variants/lib_$v.so timeout 600 python tools/kernel_bench.py --reps 12 --only gatherrows --modes $M > $O/kbg_$v.json 2> $O/kbg_$v.txt
done
tail -3 $O/pytest.log; for v in now3 cm0; do echo "== $v"; cat $O/kb_$v.txt; done; for v in now3 cs cs_nosw live; do echo "== $v"; cat $O/kbg_$v.txt; done
