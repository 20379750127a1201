#!/bin/bash
cd "$(dirname "$0")/.."
O=gpurun_out/r02it2; mkdir -p $O
timeout 1500 python -m pytest -q -p no:cacheprovider -m gpu -x tests/test_gpu_scatter_bucketed.py tests/test_gpu_kernels.py tests/test_gpu_count_modes.py tests/test_gpu_modulo.py tests/test_gpu_fuzz.py tests/test_gpu_fullscale.py -k "scatter or stencil or gather" > $O/pytest.log 2>&1
echo "rc=$?" >> $O/pytest.log
GD_CHECK_PER_ACCESS=1 timeout 900 python -m pytest -q -p no:cacheprovider -m gpu -x tests/test_gpu_kernels.py tests/test_gpu_count_modes.py tests/test_gpu_modulo.py tests/test_gpu_fuzz.py -k "stencil or gather" > $O/pytest_pa.log 2>&1
echo "rc=$?" >> $O/pytest_pa.log
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:k_stencil_pa" -s 1 -c 1 -o $O/st_check_pa -f python tools/prof_kernel.py --kind stencil --mode check --pa --reps 2 > $O/ncu1.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:k_stencil" -s 1 -c 1 -o $O/st_none -f python tools/prof_kernel.py --kind stencil --mode none --reps 2 > $O/ncu2.log 2>&1
M=none,mask,check,modulo,maskcount,clamp,check+pa,modulo+pa,maskcount+pa,clamp+pa
timeout 900 python tools/kernel_bench.py --reps 10 --only stencil,l2,scatter,gatherrows --modes $M > $O/kb.json 2> $O/kb.txt
tail -3 $O/pytest.log; tail -3 $O/pytest_pa.log; cat $O/kb.txt
