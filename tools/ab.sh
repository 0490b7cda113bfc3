# A/B: default libcrsh.so vs alternatives in build/ab/ (CRSH_LIB_PATH)
for v in base r72; do
  if [ $v = base ]; then L=""; else L="$PWD/build/ab/libcrsh_$v.so"; fi
  for z in "" "--zorder"; do
    CRSH_LIB_PATH=$L python bench.py --no-cpu-baseline --steps 10 $z > gpurun_out/ab_${v}${z}.log 2>&1
  done
done
