#!/bin/bash
# D = 1 gather: check / mask-count table fence on >= 4 GiB partitions as one
# LOP3 (Fence::in_big) with bit-mask counting; gather parity hoisted and per
# access, kernel bench (HBM + L2 gathers) and one bench.py run, new vs head.
cd "$(dirname "$0")/.."
O=gpurun_out/r02it26; mkdir -p $O
timeout 900 python -m pytest -q -p no:cacheprovider -m gpu tests -k "gather" > $O/pytest.log 2>&1
echo "rc=$?" >> $O/pytest.log
GD_CHECK_PER_ACCESS=1 timeout 900 python -m pytest -q -p no:cacheprovider -m gpu tests -k "gather" > $O/pytest_pa.log 2>&1
echo "rc=$?" >> $O/pytest_pa.log
M=none,mask,check,modulo,maskcount,clamp,check+pa,modulo+pa,maskcount+pa,clamp+pa
for r in 1 2; do for v in g1big head; do
  GD_LIB=tools/variants/lib_$v.so timeout 900 python tools/kernel_bench.py --reps 12 --only gather,l2 --modes $M > $O/kb_${v}_$r.json 2> $O/kb_${v}_$r.txt
done; done
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err
tail -n2 $O/pytest.log; tail -n2 $O/pytest_pa.log; for v in g1big head; do echo "== $v"; grep -h "gather" $O/kb_${v}_*.txt; done
python -c "
import json;d=json.loads(open('$O/bench.json').read().strip().splitlines()[-1]);print(d['value'], d['parity']);print({k:{m:x.get('overhead_pct') for m,x in v.items()} for k,v in d['l2_resident_per_access'].items() if 'gather' in k})"
