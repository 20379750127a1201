#!/bin/bash
# Round-2 iteration: scatter (bucketed) + stencil parity, hoisted and per access; kernel bench.
cd "$(dirname "$0")/.."
O=gpurun_out/r02it; mkdir -p $O
timeout 1200 python -m pytest -q -p no:cacheprovider -m gpu -x tests/test_gpu_scatter_bucketed.py tests/test_gpu_kernels.py tests/test_gpu_count_modes.py tests/test_gpu_modulo.py tests/test_gpu_fuzz.py tests/test_gpu_fullscale.py -k "scatter or stencil or c2" > $O/pytest.log 2>&1
echo "rc=$?" >> $O/pytest.log
GD_CHECK_PER_ACCESS=1 timeout 900 python -m pytest -q -p no:cacheprovider -m gpu -x tests/test_gpu_kernels.py tests/test_gpu_count_modes.py tests/test_gpu_modulo.py tests/test_gpu_fuzz.py -k "stencil and not v2" > $O/pytest_pa.log 2>&1
echo "rc=$?" >> $O/pytest_pa.log
M=none,mask,check,modulo,maskcount,clamp,check+pa,modulo+pa,maskcount+pa,clamp+pa
timeout 900 python tools/kernel_bench.py --reps 10 --only stencil,l2,scatter,gatherrows --modes $M > $O/kb.json 2> $O/kb.txt
GD_SCATTER_DIRECT=1 timeout 600 python tools/kernel_bench.py --reps 6 --only scatter --modes none,mask,check > $O/kb_direct.json 2> $O/kb_direct.txt
tail -3 $O/pytest.log; tail -3 $O/pytest_pa.log; cat $O/kb.txt $O/kb_direct.txt
