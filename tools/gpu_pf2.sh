# prefilter per hash (child only for R6, child + top level for Z-order): full GPU suite on the build, then A/B vs the child-only build
CRSH_LIB_PATH=$PWD/build/ab/libcrsh_pf2.so timeout 1500 python -m pytest tests -m gpu -q -x -k "not bench_contract" > gpurun_out/pf2_tests.log 2>&1; tail -3 gpurun_out/pf2_tests.log
bash tools/ab_trav.sh "4 3 2" "--zorder, " pf1 pf2 2>/dev/null
