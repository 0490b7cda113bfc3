# GPU suite, then the compress / decompress tile A/B (env switches, same build)
python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests.log 2>&1; echo "rc=$?" >> gpurun_out/gpu_tests.log; tail -3 gpurun_out/gpu_tests.log
for v in "0 0" "1 0" "1 1" "0 1"; do
  set -- $v; export CRSH_BIG_TILES=$1 CRSH_RLE_HIST=$2
  for c in 2 4; do
    python bench.py --config $c --zorder --single-hash --no-cpu-baseline --steps 5 > gpurun_out/tl_$1$2_c$c.json 2>/dev/null
    python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[1], d['value'], d['roofline']['hbm_stages']['ms'], {k: v for k, v in d['stage_ms'].items() if k != 'traverse+final'})" gpurun_out/tl_$1$2_c$c.json
  done
done
