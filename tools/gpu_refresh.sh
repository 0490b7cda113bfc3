# Round evidence refresh on the GPU box (gpurun): GPU tests, bench lines, launch lists, ncu captures.
set -x
python -m pytest tests -m gpu -q > gpurun_out/gpu_tests.log 2>&1; tail -2 gpurun_out/gpu_tests.log
python bench.py > gpurun_out/r1_bench_cfg2_R6.jsonl 2> gpurun_out/bench_err.log
python bench.py --zorder --no-cpu-baseline > gpurun_out/r1_bench_cfg2_zorder.jsonl 2>> gpurun_out/bench_err.log
python bench.py --config 3 --no-cpu-baseline > gpurun_out/r1_bench_cfg3_R6.jsonl 2>> gpurun_out/bench_err.log
python bench.py --config 3 --zorder --no-cpu-baseline > gpurun_out/r1_bench_cfg3_zorder.jsonl 2>> gpurun_out/bench_err.log
python bench.py --config 4 --no-cpu-baseline --steps 5 > gpurun_out/r1_bench_cfg4_R6.jsonl 2>> gpurun_out/bench_err.log
python bench.py --config 4 --zorder --no-cpu-baseline > gpurun_out/r1_bench_cfg4_zorder.jsonl 2>> gpurun_out/bench_err.log
python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/r1_bench_reference.jsonl 2>> gpurun_out/bench_err.log
bash tools/gpu_prof.sh
python bench.py --table4 --steps 5 > gpurun_out/r1_table4_cfg2.json 2>> gpurun_out/bench_err.log
python bench.py --table4 --steps 3 --config 3 > gpurun_out/r1_table4_cfg3.json 2>> gpurun_out/bench_err.log
