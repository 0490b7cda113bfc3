python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests.log 2>&1; echo "rc=$?" >> gpurun_out/gpu_tests.log; tail -3 gpurun_out/gpu_tests.log
bash tools/ab_trav.sh "2 3 4" "--zorder --objtree,--zorder, " ot4 sp 2>/dev/null
bash tools/ab_stages.sh ot4 sp 2>/dev/null
