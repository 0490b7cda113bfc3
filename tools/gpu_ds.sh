# A/B: slices of an item handed out by a shared counter (CRSH_DYN_SLICE)
CRSH_LIB_PATH=$PWD/build/ab/libcrsh_ds1.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_headline.py -q -x -k "cfg1 or micro or option or cfg2_full or edge or alternative or objtree or headline_full_frame_parity and 3-7" > gpurun_out/ds_par.log 2>&1; tail -2 gpurun_out/ds_par.log
bash tools/ab_trav.sh "4 3" "--zorder, ,--zorder --objtree" ds0 ds1 2>/dev/null
