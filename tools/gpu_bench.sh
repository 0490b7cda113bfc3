# bench lines on the GPU box (gpurun): default (cfg4), reference arm, cfg2/cfg3.
set -x
python bench.py > gpurun_out/bench_cfg4.jsonl 2> gpurun_out/bench_err.log; tail -c 3000 gpurun_out/bench_err.log
python bench.py --config 3 --no-cpu-baseline > gpurun_out/bench_cfg3.jsonl 2>> gpurun_out/bench_err.log
python bench.py --config 2 --no-cpu-baseline > gpurun_out/bench_cfg2.jsonl 2>> gpurun_out/bench_err.log
python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/bench_ref.jsonl 2>> gpurun_out/bench_err.log
cat gpurun_out/bench_cfg4.jsonl | head -c 4000
