# A/B: child tests unrolled over compile-time top nodes (CRSH_CHILD_UNROLL); stage yardsticks
python tools/stage_yardsticks.py --config 4 > gpurun_out/r2_stage_yardsticks_cfg4_R6.json 2> gpurun_out/ys_err.log; tail -c 1500 gpurun_out/r2_stage_yardsticks_cfg4_R6.json gpurun_out/ys_err.log
python tools/stage_yardsticks.py --config 4 --zorder > gpurun_out/r2_stage_yardsticks_cfg4_zorder.json 2>> gpurun_out/ys_err.log
bash tools/ab_trav.sh "4 3" "--zorder, " cu0 cu1 2>/dev/null
