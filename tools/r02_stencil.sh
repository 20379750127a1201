#!/bin/bash
# Round-2 stencil iteration: parity of every stencil test (hoisted and per
# access), then the six modes hoisted and per access at HBM and L2 sizes.
cd "$(dirname "$0")/.."
O=gpurun_out/r02st; mkdir -p $O
timeout 900 python -m pytest -q -p no:cacheprovider -m gpu -x tests/test_gpu_kernels.py tests/test_gpu_count_modes.py tests/test_gpu_modulo.py tests/test_gpu_fuzz.py -k "stencil" > $O/pytest.log 2>&1
echo "rc=$?" >> $O/pytest.log
GD_CHECK_PER_ACCESS=1 timeout 900 python -m pytest -q -p no:cacheprovider -m gpu -x tests/test_gpu_kernels.py tests/test_gpu_count_modes.py tests/test_gpu_modulo.py tests/test_gpu_fuzz.py tests/test_gpu_fullscale.py -k "stencil and not v2" > $O/pytest_pa.log 2>&1
echo "rc=$?" >> $O/pytest_pa.log
M=none,mask,check,modulo,maskcount,clamp,check+pa,modulo+pa,maskcount+pa,clamp+pa
timeout 900 python tools/kernel_bench.py --reps 10 --only stencil,l2 --modes $M > $O/kb.json 2> $O/kb.txt
tail -2 $O/pytest.log $O/pytest_pa.log; cat $O/kb.txt
