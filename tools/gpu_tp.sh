# A/B: K8 top-level prefilter (CRSH_TOP_PREFILTER=0|1, same build)
CRSH_TOP_PREFILTER=1 CRSH_LIB_PATH=$PWD/build/ab/libcrsh_tp.so timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_headline.py -q -x -k "prefilter or cfg1 or micro or option or cfg2_full or edge or headline_full_frame_parity and 3-7" > gpurun_out/tp_par.log 2>&1; tail -3 gpurun_out/tp_par.log
for t in 0 1; do echo "top_pf $t"; CRSH_TOP_PREFILTER=$t bash tools/ab_trav.sh "4 3 2" "--zorder, " tp 2>/dev/null; done
