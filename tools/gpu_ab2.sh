bash tools/ab_stages.sh s3 s4 s20 2>/dev/null
for it in default 4096 8192; do
  if [ $it = default ]; then unset CRSH_ITEM_TRIS; else export CRSH_ITEM_TRIS=$it; fi
  python bench.py --config 2 --zorder --objtree --single-hash --no-cpu-baseline --steps 10 > gpurun_out/it_${it}_c2.json 2>/dev/null
  python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[1], d['value'], d['ms_per_step'])" gpurun_out/it_${it}_c2.json
done
