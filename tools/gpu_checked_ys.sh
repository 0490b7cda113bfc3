# checked build on the final tree, then the stage yardsticks (library gathers included)
bash tools/gpu_checked.sh
python tools/stage_yardsticks.py --config 4 > gpurun_out/r2_stage_yardsticks_cfg4_R6.json 2> gpurun_out/ys_err.log
python tools/stage_yardsticks.py --config 4 --zorder > gpurun_out/r2_stage_yardsticks_cfg4_zorder.json 2>> gpurun_out/ys_err.log
tail -c 600 gpurun_out/r2_stage_yardsticks_cfg4_R6.json gpurun_out/ys_err.log
