# A/B: object-tree two-phase items (CRSH_OBJ_TWOPHASE)
CRSH_LIB_PATH=$PWD/build/ab/libcrsh_op1.so timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_headline.py -q -x -k "objtree or cluster_list or option or edge or headline_full_frame_parity and 3-71" > gpurun_out/op_par.log 2>&1; tail -2 gpurun_out/op_par.log
bash tools/ab_trav.sh "4 3 2" "--zorder --objtree" op0 op1 2>/dev/null
