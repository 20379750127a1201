cd /root/repo
for m in none check; do
 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_gatherR -s 1 -c 1 -o gpurun_out/prof_rows32_$m -f python tools/prof_kernel.py --kind gatherrows --D 32 --mode $m --reps 2 > gpurun_out/ncu_rows32_$m.log 2>&1; tail -2 gpurun_out/ncu_rows32_$m.log
done
