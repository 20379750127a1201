#!/bin/bash
# Row gather clamp: the fix-up of outside vectors behind one branch, its edge
# words from a below-the-base bit per vector instead of the vectors' addresses
# (GD_GATHER_CLAMP_BITS / FIX_BRANCH bit G); parity, then D = 64 / 128.
cd "$(dirname "$0")/.."
O=gpurun_out/r02it28; mkdir -p $O
GD_LIB=tools/variants/lib_b14f14.so timeout 900 python -m pytest -q -p no:cacheprovider -m gpu tests -k "gather_rows or row_gather" > $O/pytest.log 2>&1
echo "rc=$?" >> $O/pytest.log
GD_LIB=tools/variants/lib_b14f14.so GD_CHECK_PER_ACCESS=1 timeout 900 python -m pytest -q -p no:cacheprovider -m gpu tests -k "gather_rows or row_gather" > $O/pytest_pa.log 2>&1
echo "rc=$?" >> $O/pytest_pa.log
M=none,mask,clamp,check+pa,clamp+pa
for r in 1 2; do for v in cbase b4f4 b14f14; do
  GD_LIB=tools/variants/lib_$v.so KB_D=64,128 timeout 900 python tools/kernel_bench.py --reps 12 --only gatherrows --modes $M > $O/kb_${v}_$r.json 2> $O/kb_${v}_$r.txt
done; done
tail -n2 $O/pytest.log; tail -n2 $O/pytest_pa.log; for v in cbase b4f4 b14f14; do echo "== $v"; grep -h "gather rows" $O/kb_${v}_*.txt; done
