# the GPU suite twice more and smoke, to catch flaky tests before the driver's round-end run
for i in 1 2; do python -m pytest tests -m gpu -q -p no:randomly > gpurun_out/stab_$i.log 2>&1; echo "run $i rc=$?"; tail -1 gpurun_out/stab_$i.log; done
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
