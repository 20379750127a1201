#!/bin/bash
# k_gatherE: modulo stream walk (Fence::step_up on the index and output
# streams) in 4-word passes; gather parity hoisted and per access, then
# D = 6 in ten modes, walk vs the previous build (head).
cd "$(dirname "$0")/.."
O=gpurun_out/r02it23; mkdir -p $O
timeout 900 python -m pytest -q -p no:cacheprovider -m gpu tests -k "gather" > $O/pytest.log 2>&1
echo "rc=$?" >> $O/pytest.log
GD_CHECK_PER_ACCESS=1 timeout 900 python -m pytest -q -p no:cacheprovider -m gpu tests -k "gather" > $O/pytest_pa.log 2>&1
echo "rc=$?" >> $O/pytest_pa.log
M=none,mask,check,modulo,maskcount,clamp,check+pa,modulo+pa,maskcount+pa,clamp+pa
for r in 1 2; do for v in walk head; do
  GD_LIB=tools/variants/lib_$v.so KB_D=6 timeout 900 python tools/kernel_bench.py --reps 12 --only gatherrows --modes $M > $O/kb_${v}_$r.json 2> $O/kb_${v}_$r.txt
done; done
tail -n2 $O/pytest.log; tail -n2 $O/pytest_pa.log; for v in walk head; do echo "== $v"; grep -h "D=6" $O/kb_${v}_*.txt; done
