#!/bin/bash
# A/B: hoisted stencil with the unfenced body not inlined (now5 vs nl0), and
# the modulo walk of copy / saxpy per access (now5 vs now4).
cd "$(dirname "$0")/.."
O=gpurun_out/r02it6; mkdir -p $O
timeout 900 python -m pytest -q -p no:cacheprovider -m gpu -x tests/test_gpu_kernels.py tests/test_gpu_modulo.py tests/test_gpu_peraccess.py tests/test_gpu_count_modes.py -k "stencil or copy or saxpy or modulo" > $O/pytest.log 2>&1
echo "rc=$?" >> $O/pytest.log
M=none,mask,check,modulo,maskcount,clamp,check+pa,modulo+pa,maskcount+pa,clamp+pa
for v in now5 nl0 now4; do
  GD_LIB=tools/variants/lib_$v.so timeout 600 python tools/kernel_bench.py --reps 12 --only copy,saxpy,stencil,l2 --modes $M > $O/kb_$v.json 2> $O/kb_$v.txt
done
tail -3 $O/pytest.log; for v in now5 nl0 now4; do echo "== $v"; cat $O/kb_$v.txt; done
