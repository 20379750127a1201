#!/bin/bash
# The whole GPU suite, then the whole suite again with per-access fencing,
# then the ncu captures of r02_ncu2.sh.
cd "$(dirname "$0")/.."
O=gpurun_out/r02suite; mkdir -p $O
timeout 1500 python -m pytest -q -p no:cacheprovider -m gpu tests --durations=10 > $O/pytest.log 2>&1
echo "rc=$?" >> $O/pytest.log
GD_CHECK_PER_ACCESS=1 timeout 1500 python -m pytest -q -p no:cacheprovider -m gpu tests --durations=5 > $O/pytest_pa.log 2>&1
echo "rc=$?" >> $O/pytest_pa.log
tail -4 $O/pytest.log; tail -4 $O/pytest_pa.log
bash tools/r02_ncu2.sh
