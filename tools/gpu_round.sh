#!/bin/bash
# One GPU call: tests, smoke, bench, ncu launch list.  Output under gpurun_out/.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,memory.total,clocks.max.sm,clocks.sm --format=csv > gpurun_out/gpuinfo.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider --ignore=tests/test_gpu_gemm.py ${PYTEST_ARGS} > gpurun_out/gpu_tests.log 2>&1
timeout 600 python -m pytest tests/test_gpu_gemm.py -m gpu -q -p no:cacheprovider -x > gpurun_out/gpu_gemm.log 2>&1; echo "gemm rc=$?" >> gpurun_out/gpu_gemm.log
echo "pytest rc=$?" >> gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
if [ -z "$SKIP_BENCH" ]; then
  timeout 900 python bench.py ${BENCH_ARGS} > gpurun_out/bench.json 2> gpurun_out/bench.err
  echo "bench rc=$?" >> gpurun_out/bench.err
fi
if [ -n "$NCU" ]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k 'regex:^k_' --csv \
     --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --reps 1 --no-e2e --no-cpu \
     > gpurun_out/ncu_bench.out 2>&1
  echo "ncu rc=$?" >> gpurun_out/ncu_bench.out
fi
tail -3 gpurun_out/gpu_tests.log; tail -3 gpurun_out/gpu_gemm.log; tail -2 gpurun_out/smoke.log; head -c 600 gpurun_out/bench.json; tail -2 gpurun_out/bench.err
