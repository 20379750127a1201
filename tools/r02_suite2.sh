#!/bin/bash
# The whole GPU suite of the final build, hoisted and per access, smoke, and
# the reference arm's JSON line.
cd "$(dirname "$0")/.."
O=gpurun_out/r02suite2; mkdir -p $O
timeout 1500 python -m pytest -q -p no:cacheprovider -m gpu tests --durations=10 > $O/pytest.log 2>&1
echo "rc=$?" >> $O/pytest.log
GD_CHECK_PER_ACCESS=1 timeout 1500 python -m pytest -q -p no:cacheprovider -m gpu tests --durations=5 > $O/pytest_pa.log 2>&1
echo "rc=$?" >> $O/pytest_pa.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
echo "smoke rc=$?" >> $O/smoke.log
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > $O/reference.json 2> $O/reference.err
echo "reference rc=$?" >> $O/reference.err
tail -n3 $O/pytest.log; tail -n3 $O/pytest_pa.log; cat $O/smoke.log; head -c 600 $O/reference.json; tail -n1 $O/reference.err
