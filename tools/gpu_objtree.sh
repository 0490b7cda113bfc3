python -m pytest tests -m gpu -q -x --durations=8 > gpurun_out/gpu_tests.log 2>&1; echo "rc=$?" >> gpurun_out/gpu_tests.log; tail -14 gpurun_out/gpu_tests.log
for c in 2 3 4; do for z in "" "--zorder"; do for o in "" "--objtree"; do
python bench.py --config $c $z $o --single-hash --no-cpu-baseline --steps 5 > gpurun_out/ot_c${c}${z}${o}.json 2>/dev/null
python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[1], d['value'], d['ms_per_step'], d['tests_per_ray'], d['roofline']['frac'], d['stage_ms']['traverse+final'])" gpurun_out/ot_c${c}${z}${o}.json
done; done; done
