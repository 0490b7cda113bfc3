# Checked build (device bounds checks, -DCRSH_CHECKED=1; the memcheck stand-in while compute-sanitizer
# is closed on this pool): the GPU suite with the graph, then the parity files with direct launches.
L=$PWD/build/ab/libcrsh_checked.so
CRSH_LIB_PATH=$L python -m pytest tests -m gpu -q -x -k "not bench_contract" > gpurun_out/checked_graph.log 2>&1; echo "rc=$?" >> gpurun_out/checked_graph.log
CRSH_NO_GRAPH=1 CRSH_LIB_PATH=$L python -m pytest tests/test_gpu_parity.py tests/test_gpu_two_process.py tests/test_gpu_dist.py -q -x > gpurun_out/checked_nograph.log 2>&1; echo "rc=$?" >> gpurun_out/checked_nograph.log
tail -n 3 gpurun_out/checked_graph.log gpurun_out/checked_nograph.log
