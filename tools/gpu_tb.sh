python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; tail -2 gpurun_out/gpu_tests.log
python bench.py --no-cpu-baseline --steps 10 > gpurun_out/bench_a.log 2>&1
python bench.py --no-cpu-baseline --steps 10 --zorder > gpurun_out/bench_a_z.log 2>&1
