# final round evidence on the GPU box
set -x
python -m pytest tests -m gpu -q --durations=8 > gpurun_out/r2_gpu_tests_final.log 2>&1; echo "rc=$?" >> gpurun_out/r2_gpu_tests_final.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke_final.log 2>&1; echo "rc=$?" >> gpurun_out/r2_smoke_final.log
python bench.py > gpurun_out/r2_bench_cfg4.jsonl 2> gpurun_out/bench_err.log
python bench.py --config 3 --no-cpu-baseline > gpurun_out/r2_bench_cfg3.jsonl 2>> gpurun_out/bench_err.log
python bench.py --config 2 --no-cpu-baseline > gpurun_out/r2_bench_cfg2.jsonl 2>> gpurun_out/bench_err.log
python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r2_bench_reference.jsonl 2>> gpurun_out/bench_err.log
python bench.py --table4 --steps 5 --config 2 > gpurun_out/r2_table4_cfg2.json 2>> gpurun_out/bench_err.log
python bench.py --table4 --steps 3 --config 3 > gpurun_out/r2_table4_cfg3.json 2>> gpurun_out/bench_err.log
python bench.py --whitted 3 --zorder --steps 5 --config 2 > gpurun_out/r2_whitted_cfg2_d3_zorder.jsonl 2>> gpurun_out/bench_err.log
python bench.py --animate 20 --zorder --config 2 > gpurun_out/r2_animate_cfg2_zorder.jsonl 2>> gpurun_out/bench_err.log
python bench.py --config 4 --zorder --single-hash --no-cpu-baseline --steps 2 --warmup 3 > gpurun_out/plain_l.log 2>&1 &&
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r2_launches_cfg4_zorder.csv python bench.py --config 4 --zorder --single-hash --no-cpu-baseline --steps 2 --warmup 3 > /dev/null 2>&1
python tools/launch_table.py gpurun_out/r2_launches_cfg4_zorder.csv > gpurun_out/r2_launch_table_cfg4_zorder.txt 2>&1
tail -4 gpurun_out/r2_gpu_tests_final.log; cat gpurun_out/r2_launch_table_cfg4_zorder.txt | head -30
