#!/bin/bash
# A/B: modulo fence fast path (offset < 2 size: one conditional subtract) --
# mf1 (on) vs mf0 (the reciprocal for every access); modulo parity first.
cd "$(dirname "$0")/.."
O=gpurun_out/r02it12; mkdir -p $O
GD_LIB=tools/variants/lib_mf1.so timeout 1200 python -m pytest -q -p no:cacheprovider -m gpu -x tests -k "modulo" > $O/pytest.log 2>&1
echo "rc=$?" >> $O/pytest.log
GD_LIB=tools/variants/lib_mf1.so GD_CHECK_PER_ACCESS=1 timeout 1200 python -m pytest -q -p no:cacheprovider -m gpu -x tests -k "modulo" > $O/pytest_pa.log 2>&1
echo "rc=$?" >> $O/pytest_pa.log
M=none,mask,modulo,modulo+pa
for v in mf1 mf0; do
  GD_LIB=tools/variants/lib_$v.so timeout 900 python tools/kernel_bench.py --reps 12 --only copy,saxpy,gather,scatter,gatherrows,stencil,l2 --modes $M > $O/kb_$v.json 2> $O/kb_$v.txt
done
tail -2 $O/pytest.log; tail -2 $O/pytest_pa.log; for v in mf1 mf0; do echo "== $v"; cat $O/kb_$v.txt; done
