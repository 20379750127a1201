#!/bin/bash
# A/B: scatter-add v2 with branch-free stream loads and the modulo stream
# walk (now7) vs before (now6); scatter parity first.
cd "$(dirname "$0")/.."
O=gpurun_out/r02it9; mkdir -p $O
timeout 1200 python -m pytest -q -p no:cacheprovider -m gpu -x tests -k "scatter" > $O/pytest.log 2>&1
echo "rc=$?" >> $O/pytest.log
GD_CHECK_PER_ACCESS=1 timeout 1200 python -m pytest -q -p no:cacheprovider -m gpu -x tests -k "scatter" > $O/pytest_pa.log 2>&1
echo "rc=$?" >> $O/pytest_pa.log
M=none,mask,check,modulo,maskcount,clamp,check+pa,modulo+pa,maskcount+pa,clamp+pa
for v in now8 now6; do
  GD_LIB=tools/variants/lib_$v.so timeout 600 python tools/kernel_bench.py --reps 12 --only scatter --modes $M > $O/kb_$v.json 2> $O/kb_$v.txt
done
tail -3 $O/pytest.log; tail -3 $O/pytest_pa.log; for v in now8 now6; do echo "== $v"; cat $O/kb_$v.txt; done
