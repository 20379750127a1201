cd /root/repo; O=gpurun_out/r02l2g; mkdir -p $O
for k in bench_ws plain; do for m in none check+pa; do
  timeout 600 ncu --set full --cache-control none --clock-control none --kernel-name-base demangled -k "regex:k_gather1<" -s 2 -c 1 -o $O/${k}_${m} -f python tools/l2_gather_probe.py $k --once $m > $O/${k}_$m.log 2>&1
  mv -f $O/_$m.ncu-rep $O/${k}_${m}.ncu-rep 2>/dev/null
done; done
python tools/ncu_summary.py $O/*.ncu-rep --out $O/sum.json --traffic $O/t.json > $O/sum.txt 2>&1
rm -f $O/*.ncu-rep; ls $O
