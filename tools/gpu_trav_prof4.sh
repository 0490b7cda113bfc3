# k_traverse ncu --set full at cfg4 (R6; Z-order; Z-order + object tree), child-prefilter tree, exported to CSV on the box
for v in "r6:" "z:--zorder" "zot:--zorder --objtree"; do
  n=${v%%:*}; f=${v#*:}
  python bench.py --config 4 $f --single-hash --no-cpu-baseline --steps 1 --warmup 3 > gpurun_out/plain_$n.log 2>&1 &&
  ncu --set full --clock-control none --import-source on -k regex:k_traverse -s 3 -c 1 -o /tmp/trav_c4_$n -f \
    python bench.py --config 4 $f --single-hash --no-cpu-baseline --steps 1 --warmup 3 > gpurun_out/ncu_$n.log 2>&1
  ncu -i /tmp/trav_c4_$n.ncu-rep --page raw --csv > gpurun_out/trav4_c4_${n}_raw.csv 2>/dev/null
  ncu -i /tmp/trav_c4_$n.ncu-rep --page source --csv --print-source sass > gpurun_out/trav4_c4_${n}_sass.csv 2>/dev/null
  gzip -f gpurun_out/trav4_c4_${n}_sass.csv
done
ls -la gpurun_out
