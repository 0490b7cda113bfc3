# confirm the final binary: the GPU suite, smoke, the default bench line
python -m pytest tests -m gpu -q > gpurun_out/confirm_tests.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/confirm_tests.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
python bench.py > gpurun_out/confirm_bench.jsonl 2> gpurun_out/confirm_bench.err; echo "bench rc=$?"
python -c "import json; d=json.loads(open('gpurun_out/confirm_bench.jsonl').readline()); print(d['value'], d['value_zorder'], d['value_zorder_objtree'], d['roofline']['frac'], d['e2e']['value'], d['clocks'])"
