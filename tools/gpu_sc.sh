CRSH_LIB_PATH=$PWD/build/ab/libcrsh_sc96.so python -m pytest tests/test_gpu_parity.py tests/test_gpu_headline.py -q -x -k "cfg2_full or 3-7 or 4-7 or 3-3" > gpurun_out/sc_par.log 2>&1; tail -2 gpurun_out/sc_par.log
bash tools/ab_trav.sh "2 3 4" "--zorder, " sc0 sc32 sc96 sc256 2>/dev/null
