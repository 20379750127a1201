#!/bin/bash
# Round-2 state check of HEAD: the whole GPU suite, smoke, the bench line,
# and the kernel bench of every kernel hoisted and per access.
cd "$(dirname "$0")/.."
O=gpurun_out/r02state; mkdir -p $O
nvidia-smi --query-gpu=name,memory.total,clocks.max.sm,clocks.sm,power.limit --format=csv > $O/gpuinfo.txt 2>&1
timeout 2400 python -m pytest -q -p no:cacheprovider -m gpu tests --durations=20 ${PYTEST_ARGS} > $O/pytest.log 2>&1
echo "rc=$?" >> $O/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
echo "smoke rc=$?" >> $O/smoke.log
timeout 1200 python bench.py > $O/bench.json 2> $O/bench.err
echo "bench rc=$?" >> $O/bench.err
M=none,mask,check,modulo,maskcount,clamp,check+pa,modulo+pa,maskcount+pa,clamp+pa
timeout 1500 python tools/kernel_bench.py --reps 10 --only copy,saxpy,gather,scatter,gatherrows,stencil,stencil_tma,l2,gemm --modes $M > $O/kb.json 2> $O/kb.txt
echo "kb rc=$?" >> $O/kb.txt
tail -30 $O/pytest.log; cat $O/smoke.log; head -c 800 $O/bench.json; tail -3 $O/bench.err; tail -80 $O/kb.txt
