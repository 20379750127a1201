#!/bin/bash
# A/B: zero-block redirect of refused check loads, one-LOP3 mask fence on
# >= 4 GiB partitions (stencil), vs the previous build; parity subset first.
cd "$(dirname "$0")/.."
O=gpurun_out/r02it4; mkdir -p $O
timeout 900 python -m pytest -q -p no:cacheprovider -m gpu -x tests/test_gpu_kernels.py tests/test_gpu_count_modes.py tests/test_gpu_modulo.py tests/test_gpu_peraccess.py -k "stencil or gather" > $O/pytest.log 2>&1
echo "rc=$?" >> $O/pytest.log
M=none,mask,check,maskcount,check+pa,modulo+pa,maskcount+pa,clamp+pa
for v in base now noredir_idx noredir_st; do
  GD_LIB=tools/variants/lib_$v.so timeout 600 python tools/kernel_bench.py --reps 12 --only stencil,gatherrows,l2 --modes $M > $O/kb_$v.json 2> $O/kb_$v.txt
done
tail -3 $O/pytest.log; for v in base now noredir_idx noredir_st; do echo "== $v"; cat $O/kb_$v.txt; done
