#!/bin/bash
# Round-2: whole GPU suite, smoke, the bench line, kernel bench, scatter stages.
cd "$(dirname "$0")/.."
O=gpurun_out/r02f2; mkdir -p $O
timeout 2400 python -m pytest -q -p no:cacheprovider -m gpu tests --durations=15 > $O/pytest.log 2>&1
echo "rc=$?" >> $O/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
timeout 1200 python bench.py > $O/bench.json 2> $O/bench.err
echo "bench rc=$?" >> $O/bench.err
M=none,mask,check,modulo,maskcount,clamp,check+pa,modulo+pa,maskcount+pa,clamp+pa
timeout 900 python tools/kernel_bench.py --reps 10 --only scatter,gatherrows --modes $M > $O/kb.json 2> $O/kb.txt
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed --clock-control none -k "regex:k_scatter" --csv --log-file $O/scatter_stages.csv python tools/prof_kernel.py --kind scatter --mode mask --reps 2 > $O/scatter_stages.log 2>&1
tail -25 $O/pytest.log; tail -3 $O/smoke.log; head -c 1500 $O/bench.json; tail -3 $O/bench.err; cat $O/kb.txt
