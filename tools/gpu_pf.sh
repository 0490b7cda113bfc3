# A/B: K8 child prefilter (PF instantiation; CRSH_NO_PREFILTER=1 disables it at run time)
CRSH_LIB_PATH=$PWD/build/ab/libcrsh_pf1.so timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_headline.py -q -x -k "prefilter or cfg1 or micro or option or cfg2_full or edge or alternative or objtree or headline_full_frame_parity and 3-3" > gpurun_out/pf_par.log 2>&1; tail -3 gpurun_out/pf_par.log
bash tools/ab_trav.sh "4 3" "--zorder, " cur pf1 2>/dev/null
CRSH_NO_PREFILTER=1 bash tools/ab_trav.sh "4" "--zorder, " pf1 2>/dev/null
