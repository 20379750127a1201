#!/bin/bash
# k_gatherE counting modes in 4-word passes at 6 CTAs (narrow) vs 8 words at
# 5 CTAs; direct k_scatter at 4 CTAs per SM in every mode: parity.
cd "$(dirname "$0")/.."
O=gpurun_out/r02it22; mkdir -p $O
timeout 900 python -m pytest -q -p no:cacheprovider -m gpu tests -k "scatter or gather_rows" > $O/pytest.log 2>&1
echo "rc=$?" >> $O/pytest.log
GD_LIB=tools/variants/lib_narrow.so timeout 900 python -m pytest -q -p no:cacheprovider -m gpu tests -k "gather_rows" > $O/pytest_narrow.log 2>&1
echo "rc=$?" >> $O/pytest_narrow.log
M=none,mask,check,modulo,maskcount,clamp,check+pa,modulo+pa,maskcount+pa,clamp+pa
for r in 1 2; do for v in new narrow; do
  L=""; [ $v = narrow ] && L=tools/variants/lib_narrow.so
  GD_LIB=$L KB_D=6 timeout 900 python tools/kernel_bench.py --reps 12 --only gatherrows --modes $M > $O/kb_${v}_$r.json 2> $O/kb_${v}_$r.txt
done; done
tail -2 $O/pytest.log; tail -2 $O/pytest_narrow.log; for v in new narrow; do echo "== $v"; grep -h "D=6" $O/kb_${v}_*.txt; done
