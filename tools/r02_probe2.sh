#!/bin/bash
# Round-2 probe 2: stencil (new clamp path) parity + ncu source-level captures
# of the per-access stencil (L2 size and HBM clamp) and row gather.
cd "$(dirname "$0")/.."
O=gpurun_out/r02p2; mkdir -p $O
GD_CHECK_PER_ACCESS=1 timeout 900 python -m pytest -q -p no:cacheprovider -m gpu -x tests/test_gpu_kernels.py tests/test_gpu_count_modes.py tests/test_gpu_modulo.py tests/test_gpu_fuzz.py -k "stencil and not v2" > $O/pytest_pa.log 2>&1
echo "rc=$?" >> $O/pytest_pa.log
timeout 900 python -m pytest -q -p no:cacheprovider -m gpu -x tests/test_gpu_kernels.py tests/test_gpu_count_modes.py tests/test_gpu_fuzz.py -k "stencil and not v2" > $O/pytest.log 2>&1
echo "rc=$?" >> $O/pytest.log
prof() {  # name kernel-regex args...
  local name=$1 kre=$2; shift 2
  timeout 600 ncu --set full --clock-control none --import-source on -k "regex:${kre}" -s 1 -c 1 \
      -o $O/$name -f python tools/prof_kernel.py --reps 2 "$@" > $O/$name.log 2>&1
  echo "rc=$?" >> $O/$name.log
}
prof st_l2_none k_stencil --kind stencil --mode none --l2
prof st_l2_mask k_stencil --kind stencil --mode mask --l2
prof st_l2_check_pa k_stencil_pa --kind stencil --mode check --l2 --pa
prof st_clamp_pa k_stencil_pa --kind stencil --mode clamp --pa
prof gr_check_pa k_gatherR --kind gatherrows --mode check --pa
prof gr_check k_gatherR --kind gatherrows --mode check
M=none,mask,check,modulo,maskcount,clamp,check+pa,modulo+pa,maskcount+pa,clamp+pa
timeout 900 python tools/kernel_bench.py --reps 10 --only stencil,l2 --modes $M > $O/kb.json 2> $O/kb.txt
tail -2 $O/pytest.log $O/pytest_pa.log; cat $O/kb.txt
