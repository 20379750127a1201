#!/bin/bash
# New small-grid / 16 GiB partition crossing parity (hoisted and per access);
# A/B of mask-count's BIG variant at 8-row strips (now12 vs mcb0).
cd "$(dirname "$0")/.."
O=gpurun_out/r02it14; mkdir -p $O
timeout 1200 python -m pytest -q -p no:cacheprovider -m gpu tests/test_gpu_fullscale.py -k "crossing" > $O/pytest.log 2>&1
echo "rc=$?" >> $O/pytest.log
GD_CHECK_PER_ACCESS=1 timeout 1200 python -m pytest -q -p no:cacheprovider -m gpu tests/test_gpu_fullscale.py -k "crossing" > $O/pytest_pa.log 2>&1
echo "rc=$?" >> $O/pytest_pa.log
for v in now12 mcb0; do
  GD_LIB=tools/variants/lib_$v.so timeout 900 python tools/kernel_bench.py --reps 12 --only l2 --modes none,mask,maskcount,check+pa,maskcount+pa,clamp+pa > $O/kb_$v.json 2> $O/kb_$v.txt
done
tail -3 $O/pytest.log; tail -3 $O/pytest_pa.log; for v in now12 mcb0; do echo "== $v"; grep -i "stencil 2048" $O/kb_$v.txt; done
