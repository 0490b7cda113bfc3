python -m pytest tests/test_gpu_parity.py tests/test_gpu_headline.py -q -x -k "not headline or 3-7 or 4-7" > gpurun_out/bar_par.log 2>&1; tail -2 gpurun_out/bar_par.log
bash tools/ab_trav.sh "2 3 4" "--zorder --objtree,--zorder, " bar0 bar1 2>/dev/null
