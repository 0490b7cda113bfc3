python -m pytest tests -m gpu -q -x --durations=5 > gpurun_out/gpu_tests.log 2>&1; echo "rc=$?" >> gpurun_out/gpu_tests.log; tail -9 gpurun_out/gpu_tests.log
bash tools/ab_trav.sh "2 3 4" "--zorder --objtree,--zorder, " ot3 ot4 2>/dev/null
bash tools/ab_stages.sh ot3 ot4 2>/dev/null
