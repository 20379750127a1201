#!/bin/bash
# scatter-add: near modulo (one correction instead of the reciprocal when the
# table lies in a >= 2^33-byte partition): scatter parity hoisted and per
# access (incl. the 8 GiB + 14 MiB exact partition), kernel bench new vs head.
cd "$(dirname "$0")/.."
O=gpurun_out/r02it27; mkdir -p $O
timeout 1200 python -m pytest -q -p no:cacheprovider -m gpu tests -k "scatter" > $O/pytest.log 2>&1
echo "rc=$?" >> $O/pytest.log
GD_CHECK_PER_ACCESS=1 timeout 1200 python -m pytest -q -p no:cacheprovider -m gpu tests -k "scatter" > $O/pytest_pa.log 2>&1
echo "rc=$?" >> $O/pytest_pa.log
M=none,mask,check,modulo,maskcount,clamp,check+pa,modulo+pa,maskcount+pa,clamp+pa
for r in 1 2; do for v in near head; do
  GD_LIB=tools/variants/lib_$v.so timeout 900 python tools/kernel_bench.py --reps 12 --only scatter --modes $M > $O/kb_${v}_$r.json 2> $O/kb_${v}_$r.txt
done; done
tail -n2 $O/pytest.log; tail -n2 $O/pytest_pa.log; grep -h "FAILED\|Error" $O/pytest.log | head -5; for v in near head; do echo "== $v"; grep -h scatter $O/kb_${v}_*.txt; done
