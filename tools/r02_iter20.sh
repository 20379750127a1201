#!/bin/bash
# Row gathers: k_gatherR at the unfenced twin's occupancy (8 CTAs / 32
# registers for mask / check / mask-count) and the flat word kernel k_gatherE
# for D % 4 != 0 (replacing the warp-per-row kernel): gather parity hoisted
# and per access, then every row width in ten modes, new build vs base.
cd "$(dirname "$0")/.."
O=gpurun_out/r02it20b; mkdir -p $O
timeout 900 python -m pytest -q -p no:cacheprovider -m gpu -x tests -k "gather" > $O/pytest.log 2>&1
echo "rc=$?" >> $O/pytest.log
GD_CHECK_PER_ACCESS=1 timeout 900 python -m pytest -q -p no:cacheprovider -m gpu -x tests -k "gather" > $O/pytest_pa.log 2>&1
echo "rc=$?" >> $O/pytest_pa.log
M=none,mask,check,modulo,maskcount,clamp,check+pa,modulo+pa,maskcount+pa,clamp+pa
for v in new base; do
  L=""; [ $v = base ] && L=tools/variants/lib_base.so
  GD_LIB=$L timeout 900 python tools/kernel_bench.py --reps 12 --only gatherrows --modes $M > $O/kb_$v.json 2> $O/kb_$v.txt
done
tail -2 $O/pytest.log; tail -2 $O/pytest_pa.log; for v in new base; do echo "== $v"; grep "gather rows" $O/kb_$v.txt; done
