#!/bin/bash
# The driver's round-end commands on one B200: smoke, then the bench line it
# records (python bench.py --gpus 1 --steps 20 --warmup 5), with wall time.
cd "$(dirname "$0")/.."
O=gpurun_out/r02driver; mkdir -p $O
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
s=$(date +%s)
timeout 1200 python bench.py --gpus 1 --steps 20 --warmup 5 > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/bench.err
e=$(date +%s); echo "wall_s $((e - s))" >> $O/bench.err
cat $O/smoke.log; tail -n2 $O/bench.err; head -c 400 $O/bench.json
