# HBM-stage evidence on the GPU box: CUB yardstick + ncu --set full of the a1-a8 kernels at cfg4 Z-order.
set -x
./tools/cub_sort_yardstick.bin > gpurun_out/cub_yardstick.json 2>&1; cat gpurun_out/cub_yardstick.json
ncu --set full --import-source on --clock-control none -k "regex:k_raygen|k_onesweep|k_leaves|k_expand|k_rle|k_scan_sizes|k_radix_hist|k_upper" -c 11 -o gpurun_out/hbm_r2 -f python bench.py --config 4 --zorder --single-hash --no-cpu-baseline --steps 1 --warmup 3 > gpurun_out/ncu_hbm.log 2>&1; tail -5 gpurun_out/ncu_hbm.log
ls -la gpurun_out
