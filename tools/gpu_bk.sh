# A/B: skipped nodes' child tests counted with one warp sum in full groups (CRSH_PF_BULK)
CRSH_LIB_PATH=$PWD/build/ab/libcrsh_bk1.so timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_headline.py -q -x -k "prefilter or cfg1 or micro or option or cfg2_full or edge or sharded or headline_full_frame_parity and 3-3" > gpurun_out/bk_par.log 2>&1; tail -3 gpurun_out/bk_par.log
bash tools/ab_trav.sh "4 3 2" "--zorder, " bk0 bk1 2>/dev/null
