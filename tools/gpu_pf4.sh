# A/B: child iterations whose node has no child pair past the prefilter end right after the counts
CRSH_LIB_PATH=$PWD/build/ab/libcrsh_pf4.so timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_headline.py -q -x -k "prefilter or cfg1 or micro or option or cfg2_full or edge or sharded or headline_full_frame_parity and 3-3" > gpurun_out/pf4_par.log 2>&1; tail -3 gpurun_out/pf4_par.log
bash tools/ab_trav.sh "4 3 2" "--zorder, " pf3 pf4 2>/dev/null
