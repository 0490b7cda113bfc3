# sort-stage A/B: stage_ms of bench diagnostics per variant, cfg2 and cfg4 (Z-order)
for v in "$@"; do
  CRSH_LIB_PATH=$PWD/build/ab/libcrsh_$v.so python bench.py --no-cpu-baseline --steps 5 --zorder > gpurun_out/abs_${v}_c2.log 2>&1
  CRSH_LIB_PATH=$PWD/build/ab/libcrsh_$v.so python bench.py --no-cpu-baseline --steps 3 --zorder --config 4 > gpurun_out/abs_${v}_c4.log 2>&1
done
