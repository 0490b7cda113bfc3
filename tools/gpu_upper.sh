bash tools/ab_stages.sh upw upt 2>/dev/null
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4z.csv python bench.py --config 4 --zorder --single-hash --no-cpu-baseline --steps 1 --warmup 3 > /dev/null 2>&1
python tools/launch_table.py gpurun_out/launches_c4z.csv 2>&1 | head -40
