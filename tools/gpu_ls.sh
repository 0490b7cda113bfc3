CRSH_LIB_PATH=$PWD/build/ab/libcrsh_ls1.so python -m pytest tests/test_gpu_parity.py -q -x -k "cfg1 or micro or option or cfg2_full or edge or alternative" > gpurun_out/ls_par.log 2>&1; tail -2 gpurun_out/ls_par.log
bash tools/ab_stages.sh ls0 ls1 2>/dev/null
