# A/B of the HBM-bound stages: stage_ms (bench diagnostics) per variant build/ab/libcrsh_<v>.so, cfg2 and cfg4 (Z-order)
for v in "$@"; do
  CRSH_LIB_PATH=$PWD/build/ab/libcrsh_$v.so python bench.py --no-cpu-baseline --single-hash --steps 10 --zorder --config 2 > gpurun_out/abs_${v}_c2.log 2>&1
  CRSH_LIB_PATH=$PWD/build/ab/libcrsh_$v.so python bench.py --no-cpu-baseline --single-hash --steps 3 --zorder --config 4 > gpurun_out/abs_${v}_c4.log 2>&1
done
for v in "$@"; do for c in c2 c4; do
  python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[2], sys.argv[3], d['value'], d['roofline']['hbm_stages']['ms'], {k: v for k, v in d['stage_ms'].items() if k != 'traverse+final'})" gpurun_out/abs_${v}_$c.log $v $c
done; done
