#!/bin/bash
# A/B: mask stencil walking fenced pointers (now6 vs mw0); host-level hoist;
# a full bench line of the current build.
cd "$(dirname "$0")/.."
O=gpurun_out/r02it7; mkdir -p $O
timeout 900 python -m pytest -q -p no:cacheprovider -m gpu -x tests/test_gpu_kernels.py tests/test_gpu_modulo.py tests/test_gpu_count_modes.py tests/test_gpu_isolation.py tests/test_gpu_graph.py -k "stencil or copy or saxpy or modulo or graph or isolation" > $O/pytest.log 2>&1
echo "rc=$?" >> $O/pytest.log
M=none,mask,check,modulo,maskcount,clamp,check+pa,modulo+pa,maskcount+pa,clamp+pa
for v in now6 mw0; do
  GD_LIB=tools/variants/lib_$v.so timeout 600 python tools/kernel_bench.py --reps 12 --only stencil,l2 --modes $M > $O/kb_$v.json 2> $O/kb_$v.txt
done
timeout 1200 python bench.py > $O/bench.json 2> $O/bench.err
echo "bench rc=$?" >> $O/bench.err
tail -3 $O/pytest.log; for v in now6 mw0; do echo "== $v"; cat $O/kb_$v.txt; done; head -c 1500 $O/bench.json; tail -3 $O/bench.err
