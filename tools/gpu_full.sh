set -x
python -m pytest tests -m gpu -q > gpurun_out/gpu_tests.log 2>&1; tail -2 gpurun_out/gpu_tests.log
python bench.py > gpurun_out/r1_bench_cfg2_R6.jsonl 2> gpurun_out/bench_err.log
python bench.py --zorder --no-cpu-baseline > gpurun_out/r1_bench_cfg2_zorder.jsonl 2>> gpurun_out/bench_err.log
python bench.py --config 3 --no-cpu-baseline > gpurun_out/r1_bench_cfg3_R6.jsonl 2>> gpurun_out/bench_err.log
python bench.py --config 3 --zorder --no-cpu-baseline > gpurun_out/r1_bench_cfg3_zorder.jsonl 2>> gpurun_out/bench_err.log
python bench.py --config 4 --no-cpu-baseline --steps 5 > gpurun_out/r1_bench_cfg4_R6.jsonl 2>> gpurun_out/bench_err.log
python bench.py --config 4 --zorder --no-cpu-baseline > gpurun_out/r1_bench_cfg4_zorder.jsonl 2>> gpurun_out/bench_err.log
python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/r1_bench_reference.jsonl 2>> gpurun_out/bench_err.log
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r1_launches_cfg2_R6.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r1_launches_cfg2_zorder.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --zorder > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_traverse -s 3 -c 1 -o gpurun_out/trav_full -f python bench.py --no-cpu-baseline --steps 2 --warmup 3 > /dev/null 2>&1
ls -la gpurun_out
python bench.py --whitted 3 --steps 5 > gpurun_out/r1_whitted_cfg2_d3.jsonl 2>> gpurun_out/bench_err.log
python bench.py --animate 20 > gpurun_out/r1_animate_cfg2_R6.jsonl 2>> gpurun_out/bench_err.log
python bench.py --table4 --steps 5 > gpurun_out/r1_table4_cfg2.json 2>> gpurun_out/bench_err.log
ncu --set full --clock-control none -k "regex:k_raygen|k_onesweep|k_leaves|k_expand|k_rle|k_unpack|k_scan_sizes|k_radix_hist" -c 11 -o gpurun_out/hbm_c4 -f python bench.py --config 4 --zorder --no-cpu-baseline --steps 1 --warmup 3 > /dev/null 2>&1
