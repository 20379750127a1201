#!/bin/bash
# full-size row gather parity (D = 32 k_gatherR, D = 6 k_gatherE), every mode
cd "$(dirname "$0")/.."
O=gpurun_out/r02it24; mkdir -p $O
timeout 1200 python -m pytest -q -p no:cacheprovider -m gpu tests/test_gpu_fullscale.py -k "row_gather_full" --durations=5 > $O/pytest.log 2>&1
echo "rc=$?" >> $O/pytest.log
tail -n 12 $O/pytest.log
