# round evidence on the GPU box: bench lines (default cfg4; cfg2, cfg3), reference arm, Table-4 analogue (cfg2, cfg3)
set -x
python bench.py > gpurun_out/r2_bench_cfg4.jsonl 2> gpurun_out/bench_err.log
python bench.py --config 3 --no-cpu-baseline > gpurun_out/r2_bench_cfg3.jsonl 2>> gpurun_out/bench_err.log
python bench.py --config 2 --no-cpu-baseline > gpurun_out/r2_bench_cfg2.jsonl 2>> gpurun_out/bench_err.log
python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r2_bench_reference.jsonl 2>> gpurun_out/bench_err.log
python bench.py --table4 --steps 5 --config 2 > gpurun_out/r2_table4_cfg2.json 2>> gpurun_out/bench_err.log
python bench.py --table4 --steps 3 --config 3 > gpurun_out/r2_table4_cfg3.json 2>> gpurun_out/bench_err.log
python -c "
import json
for f in ['r2_bench_cfg4.jsonl','r2_bench_cfg3.jsonl','r2_bench_cfg2.jsonl']:
    d=json.loads(open('gpurun_out/'+f).readline()); r=d['roofline']
    print(f, d['value'], d.get('value_zorder'), d.get('value_zorder_objtree'), r['frac'], r['frac_survey_convention'], r['hbm_stages']['frac'], r['hbm_stages']['ms'], d['e2e']['value'], d['clocks'])
"
tail -c 1500 gpurun_out/bench_err.log
