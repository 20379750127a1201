#!/bin/bash
# scatter: branch-free clamp stream loads (now9); L2-size stencil strip height 4 / 8 / 16.
cd "$(dirname "$0")/.."
O=gpurun_out/r02it10; mkdir -p $O
timeout 1200 python -m pytest -q -p no:cacheprovider -m gpu -x tests -k "scatter" > $O/pytest.log 2>&1
echo "rc=$?" >> $O/pytest.log
GD_CHECK_PER_ACCESS=1 timeout 1200 python -m pytest -q -p no:cacheprovider -m gpu -x tests -k "scatter" > $O/pytest_pa.log 2>&1
echo "rc=$?" >> $O/pytest_pa.log
M=none,mask,check,modulo,maskcount,clamp,check+pa,modulo+pa,maskcount+pa,clamp+pa
GD_LIB=tools/variants/lib_now9.so timeout 600 python tools/kernel_bench.py --reps 12 --only scatter --modes $M > $O/kb_sc.json 2> $O/kb_sc.txt
for v in now9 sr4 sr16; do
  GD_LIB=tools/variants/lib_$v.so timeout 600 python tools/kernel_bench.py --reps 12 --only l2 --modes none,mask,check+pa,modulo+pa,maskcount+pa,clamp+pa > $O/kb_$v.json 2> $O/kb_$v.txt
done
tail -3 $O/pytest.log; tail -3 $O/pytest_pa.log; cat $O/kb_sc.txt; for v in now9 sr4 sr16; do echo "== $v"; grep -i stencil $O/kb_$v.txt; done
