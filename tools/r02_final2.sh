#!/bin/bash
# Round-2 evidence of the final build (k_gatherE included) in one GPU call: the whole GPU suite
# (hoisted and per access), smoke, bench.py x 3, the ncu launch list of the
# bench, ncu --set full of every kernel (none / mask / check, per access for
# the LSU stencil and the row gather), the kernel bench of every kernel in ten
# modes.  Output in gpurun_out/r02final/.
cd "$(dirname "$0")/.."
O=${O:-gpurun_out/r02final2}; mkdir -p $O
nvidia-smi --query-gpu=name,memory.total,clocks.max.sm,clocks.sm,power.limit --format=csv > $O/gpuinfo.txt 2>&1
if [ -z "$SKIP_SUITES" ]; then
timeout 1500 python -m pytest -q -p no:cacheprovider -m gpu tests --durations=15 > $O/pytest.log 2>&1
echo "rc=$?" >> $O/pytest.log
GD_CHECK_PER_ACCESS=1 timeout 1500 python -m pytest -q -p no:cacheprovider -m gpu tests --durations=5 > $O/pytest_pa.log 2>&1
echo "rc=$?" >> $O/pytest_pa.log
fi
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
echo "smoke rc=$?" >> $O/smoke.log
for i in $(seq 1 ${BENCH_RUNS:-3}); do
  timeout 1200 python bench.py > $O/bench_$i.json 2> $O/bench_$i.err
  echo "bench rc=$?" >> $O/bench_$i.err
done
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -k 'regex:^k_' --csv \
   --log-file $O/launches.csv python bench.py --steps 2 --warmup 3 --reps 1 --no-e2e --no-cpu --no-c5 \
   > $O/ncu_bench.out 2>&1
echo "ncu rc=$?" >> $O/ncu_bench.out
cap() {  # name, kernel regex, prof_kernel args...
  local n=$1 k=$2; shift 2
  timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:$k" -s 1 -c 1 \
      -o $O/prof_$n -f python tools/prof_kernel.py --reps 2 "$@" > $O/prof_$n.log 2>&1
  echo "$n rc=$?" >> $O/prof_$n.log
}
for m in none mask check; do
  cap copy_$m k_copy --kind copy --mode $m
  cap saxpy_$m k_saxpy --kind saxpy --mode $m
  cap gather_$m "k_gather1<" --kind gather --mode $m --oob 0
  cap scatterA3_$m "k_scatter_part<.int.[0-9], .int.1>" --kind scatter --mode $m --oob 0
  cap scatterB_$m k_scatter_apply --kind scatter --mode $m --oob 0
  cap stencil_$m "k_stencil<" --kind stencil --mode $m
  cap stenciltma_$m k_stencil_tma --kind stencil_tma --mode $m
  cap gatherrows_$m k_gatherR --kind gatherrows --D 32 --mode $m
  cap gemm_$m k_gemm2 --kind gemm --mode $m
  cap gathere_$m k_gatherE --kind gatherrows --D 6 --mode $m
done
for m in check modulo maskcount clamp; do
  cap stencilpa_$m k_stencil_pa --kind stencil --mode $m --pa
  cap gatherrowspa_$m k_gatherR --kind gatherrows --D 32 --mode $m --pa
  cap gatherepa_$m k_gatherE --kind gatherrows --D 6 --mode $m --pa
done
# summarise on the box (gpurun brings back at most 64 MiB): every capture
# into one JSON, DRAM bytes + throughput per kernel into a copy of
# profiles/ncu_traffic.json; keep the .ncu-rep of the dominant kernel only
cp profiles/ncu_traffic.json $O/ncu_traffic.json
python tools/ncu_summary.py $O/prof_*.ncu-rep --out $O/ncu_full.json --traffic $O/ncu_traffic.json > $O/ncu_full.txt 2>&1
for f in $O/prof_*.ncu-rep; do case $f in *prof_saxpy_mask.ncu-rep) ;; *) rm -f $f ;; esac; done
M=none,mask,check,modulo,maskcount,clamp,check+pa,modulo+pa,maskcount+pa,clamp+pa
timeout 1500 python tools/kernel_bench.py --reps 12 --only copy,saxpy,gather,scatter,gatherrows,stencil,stencil_tma,l2,gemm --modes $M > $O/kb.json 2> $O/kb.txt
echo "kb rc=$?" >> $O/kb.txt
tail -3 $O/pytest.log; tail -3 $O/pytest_pa.log; cat $O/smoke.log; for f in $O/bench_*.json; do head -c 300 $f; echo; done; du -sh $O; tail -2 $O/ncu_bench.out; grep -h "rc=" $O/prof_*.log | sort | uniq -c | sort -rn | head; tail -30 $O/kb.txt
python tools/register_report.py --out $O/registers.json > $O/registers.txt 2>&1
