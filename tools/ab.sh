# A/B: bench each build/ab/libcrsh_<v>.so named on the command line (CRSH_LIB_PATH)
for v in "$@"; do
  for z in "" "--zorder"; do
    CRSH_LIB_PATH=$PWD/build/ab/libcrsh_$v.so python bench.py --no-cpu-baseline --steps 10 $z > gpurun_out/ab_${v}${z}.log 2>&1
  done
done
