# pixel-major raygen + warp-reduction k_upper: GPU suite, then stage A/B against the slot-major raygen (same build)
python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests.log 2>&1; echo "rc=$?" >> gpurun_out/gpu_tests.log; tail -4 gpurun_out/gpu_tests.log
for mode in slot px; do
  for c in 2 3 4; do
    if [ $mode = slot ]; then export CRSH_SLOT_MAJOR=1; else unset CRSH_SLOT_MAJOR; fi
    python bench.py --config $c --zorder --single-hash --no-cpu-baseline --steps 5 > gpurun_out/rg_${mode}_c$c.json 2>/dev/null
    python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[1], d['value'], d['roofline']['hbm_stages']['ms'], {k: v for k, v in d['stage_ms'].items() if k != 'traverse+final'})" gpurun_out/rg_${mode}_c$c.json
  done
done
