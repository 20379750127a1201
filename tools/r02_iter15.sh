#!/bin/bash
# D = 1 gather: range-only table check, one-LOP3 test on >= 4 GiB partitions
# (now13) vs now12; gather parity hoisted and per access.
cd "$(dirname "$0")/.."
O=gpurun_out/r02it15; mkdir -p $O
timeout 1200 python -m pytest -q -p no:cacheprovider -m gpu -x tests -k "gather or c1 or multitenant or smoke or isolation" > $O/pytest.log 2>&1
echo "rc=$?" >> $O/pytest.log
GD_CHECK_PER_ACCESS=1 timeout 1200 python -m pytest -q -p no:cacheprovider -m gpu -x tests -k "gather or c1" > $O/pytest_pa.log 2>&1
echo "rc=$?" >> $O/pytest_pa.log
M=none,mask,check,maskcount,clamp,check+pa,maskcount+pa,clamp+pa
for v in now13 now12; do
  GD_LIB=tools/variants/lib_$v.so timeout 900 python tools/kernel_bench.py --reps 12 --only gather,l2 --modes $M > $O/kb_$v.json 2> $O/kb_$v.txt
done
tail -2 $O/pytest.log; tail -2 $O/pytest_pa.log; for v in now13 now12; do echo "== $v"; grep -i "gather" $O/kb_$v.txt; done
