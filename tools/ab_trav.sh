# A/B of the traversal: Mrays/s, ms/frame and k_traverse frac per variant build/ab/libcrsh_<v>.so
# usage: tools/ab_trav.sh "CFGS" "EXTRA FLAG SETS (comma-separated)" variants...
cfgs=$1; sets=$2; shift 2
for v in "$@"; do for c in $cfgs; do IFS=','; for f in $sets; do IFS=' '
  out=gpurun_out/abt_${v}_c${c}_$(echo "$f" | tr -d ' -').json
  CRSH_LIB_PATH=$PWD/build/ab/libcrsh_$v.so python bench.py --config $c $f --single-hash --no-cpu-baseline --steps 5 > $out 2>/dev/null
  python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[2], sys.argv[3], sys.argv[4], d['value'], d['ms_per_step'], d['tests_per_ray'], d['roofline']['frac'])" $out $v $c "$f"
done; IFS=' '; done; done
