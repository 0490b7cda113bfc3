# GPU test suite on the box (gpurun): durations of the slowest tests included.
python -m pytest tests -m gpu -q -x --durations=15 > gpurun_out/gpu_tests.log 2>&1; echo "rc=$?" >> gpurun_out/gpu_tests.log
tail -25 gpurun_out/gpu_tests.log
