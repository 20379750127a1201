#!/bin/bash
# mask on >= 4 GiB partitions in the streaming kernels (kMaskBig, now11) vs
# before (now10); parity of copy / saxpy; ncu of k_saxpy<mask_big>.
cd "$(dirname "$0")/.."
O=gpurun_out/r02it13; mkdir -p $O
timeout 1200 python -m pytest -q -p no:cacheprovider -m gpu -x tests -k "copy or saxpy or c2 or smoke or multitenant" > $O/pytest.log 2>&1
echo "rc=$?" >> $O/pytest.log
for v in now11 now10; do
  GD_LIB=tools/variants/lib_$v.so timeout 900 python tools/kernel_bench.py --reps 12 --only copy,saxpy,l2 --modes none,mask,modulo > $O/kb_$v.json 2> $O/kb_$v.txt
done
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:k_saxpy<" -s 1 -c 1 \
    -o $O/prof_saxpy_mask -f python tools/prof_kernel.py --kind saxpy --mode mask --reps 2 > $O/prof_saxpy_mask.log 2>&1
cp profiles/ncu_traffic.json $O/ncu_traffic.json
python tools/ncu_summary.py $O/prof_saxpy_mask.ncu-rep --out $O/ncu_saxpy.json --traffic $O/ncu_traffic.json > $O/ncu_saxpy.txt 2>&1
tail -2 $O/pytest.log; for v in now11 now10; do echo "== $v"; cat $O/kb_$v.txt; done; grep -i "dram_throughput\|duration\|traffic" $O/ncu_saxpy.txt
