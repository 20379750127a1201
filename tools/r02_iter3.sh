#!/bin/bash
cd "$(dirname "$0")/.."
O=gpurun_out/r02it3; mkdir -p $O
timeout 1200 python -m pytest -q -p no:cacheprovider -m gpu -x tests/test_gpu_kernels.py tests/test_gpu_count_modes.py tests/test_gpu_modulo.py tests/test_gpu_fuzz.py tests/test_gpu_fullscale.py -k "gather" > $O/pytest.log 2>&1
echo "rc=$?" >> $O/pytest.log
GD_CHECK_PER_ACCESS=1 timeout 900 python -m pytest -q -p no:cacheprovider -m gpu -x tests/test_gpu_kernels.py tests/test_gpu_count_modes.py tests/test_gpu_modulo.py tests/test_gpu_fuzz.py -k "gather" > $O/pytest_pa.log 2>&1
echo "rc=$?" >> $O/pytest_pa.log
M=none,mask,check,modulo,maskcount,clamp,check+pa,modulo+pa,maskcount+pa,clamp+pa
timeout 900 python tools/kernel_bench.py --reps 10 --only gatherrows --modes $M > $O/kb.json 2> $O/kb.txt
for v in v1 v2; do
  GD_LIB=tools/variants/lib_$v.so timeout 600 python tools/kernel_bench.py --reps 10 --only stencil --modes none,check,check+pa,maskcount+pa,clamp+pa > $O/kb_$v.json 2> $O/kb_$v.txt
done
timeout 600 python tools/kernel_bench.py --reps 10 --only stencil --modes none,check,check+pa,maskcount+pa,clamp+pa > $O/kb_v0.json 2> $O/kb_v0.txt
tail -3 $O/pytest.log; tail -3 $O/pytest_pa.log; cat $O/kb.txt; for v in v0 v1 v2; do echo $v; cat $O/kb_$v.txt; done
