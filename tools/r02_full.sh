#!/bin/bash
# Round-2: the whole GPU suite, then the stencil / L2 kernel bench (hoisted and per access).
cd "$(dirname "$0")/.."
O=gpurun_out/r02full; mkdir -p $O
timeout 1500 python -m pytest -q -p no:cacheprovider -m gpu tests ${PYTEST_ARGS} > $O/pytest.log 2>&1
echo "rc=$?" >> $O/pytest.log
M=none,mask,check,modulo,maskcount,clamp,check+pa,modulo+pa,maskcount+pa,clamp+pa
timeout 900 python tools/kernel_bench.py --reps 10 --only stencil,l2,gatherrows --modes $M > $O/kb.json 2> $O/kb.txt
tail -15 $O/pytest.log; cat $O/kb.txt
