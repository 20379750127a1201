#!/bin/bash
# scatter-add v2 slice size 16 / 32 / 64 MiB (sl24 / sl25 / sl26) and without
# the L2 bulk prefetch (nopf); scatter parity with each.
cd "$(dirname "$0")/.."
O=gpurun_out/r02it16; mkdir -p $O
for v in sl24 sl26; do
  GD_LIB=tools/variants/lib_$v.so timeout 900 python -m pytest -q -p no:cacheprovider -m gpu -x tests -k "scatter" > $O/pytest_$v.log 2>&1
  echo "rc=$?" >> $O/pytest_$v.log
done
for v in sl25 sl24 sl26 nopf; do
  GD_LIB=tools/variants/lib_$v.so timeout 900 python tools/kernel_bench.py --reps 12 --only scatter --modes none,mask,check,modulo > $O/kb_$v.json 2> $O/kb_$v.txt
done
for v in sl24 sl26; do tail -2 $O/pytest_$v.log; done; for v in sl25 sl24 sl26 nopf; do echo "== $v"; cat $O/kb_$v.txt; done
