# Refresh the round's launch lists and ncu --set full captures (run on the GPU box via gpurun).
set -x
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_cfg2_R6.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_cfg2_zorder.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --zorder > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_traverse -s 3 -c 1 -o gpurun_out/trav_full -f python bench.py --no-cpu-baseline --steps 2 --warmup 3 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k "regex:k_raygen|k_onesweep|k_leaves|k_expand|k_rle|k_unpack|k_scan_sizes|k_radix_hist" -c 11 -o gpurun_out/hbm_c4 -f python bench.py --config 4 --zorder --no-cpu-baseline --steps 1 --warmup 3 > /dev/null 2>&1
ls -la gpurun_out
