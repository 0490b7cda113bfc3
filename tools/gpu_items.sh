python -m pytest tests/test_gpu_dist.py -q -x > gpurun_out/dist.log 2>&1; tail -2 gpurun_out/dist.log
for it in default 32768 65536; do
  if [ $it = default ]; then unset CRSH_ITEM_TRIS; else export CRSH_ITEM_TRIS=$it; fi
  for c in 3 4; do
    python bench.py --config $c --zorder --objtree --single-hash --no-cpu-baseline --steps 5 > gpurun_out/it_${it}_c$c.json 2>/dev/null
    python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[1], d['value'], d['ms_per_step'])" gpurun_out/it_${it}_c$c.json
  done
done
