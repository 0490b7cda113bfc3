# k_traverse ncu --set full captures at cfg4 (R6, Z-order, Z-order + object tree), each after a plain run
set -x
for v in "r6:" "z:--zorder" "zot:--zorder --objtree"; do
  n=${v%%:*}; f=${v#*:}
  python bench.py --config 4 $f --single-hash --no-cpu-baseline --steps 1 --warmup 3 > gpurun_out/plain_$n.log 2>&1 &&
  ncu --set full --clock-control none --import-source on -k regex:k_traverse -s 3 -c 1 -o gpurun_out/trav_c4_$n -f \
    python bench.py --config 4 $f --single-hash --no-cpu-baseline --steps 1 --warmup 3 > gpurun_out/ncu_$n.log 2>&1
  tail -2 gpurun_out/ncu_$n.log
done
ls -la gpurun_out/*.ncu-rep
