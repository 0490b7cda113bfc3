# the GPU suite on the product build, then on the checked build (graph + direct launches)
python -m pytest tests -m gpu -q -x --durations=5 > gpurun_out/gpu_tests.log 2>&1; echo "rc=$?" >> gpurun_out/gpu_tests.log; tail -9 gpurun_out/gpu_tests.log
bash tools/gpu_checked.sh
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log; tail -2 gpurun_out/smoke.log
