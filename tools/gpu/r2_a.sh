# round 2, first validation: GPU suite, smoke, c2 step in both arithmetics, bench
timeout 1800 python -m pytest tests -m gpu -q -rs > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -25 gpurun_out/pytest_gpu.log | grep -E "passed|failed|FAILED|Error|drift"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 300 python tools/kstats_c2.py 2>&1 | tail -1
PINT_ARITH=exact timeout 300 python tools/kstats_c2.py 2>&1 | tail -1
timeout 900 python bench.py --no-cpu > gpurun_out/bench.jsonl 2> gpurun_out/bench.err; echo "bench rc=$?"
tail -3 gpurun_out/bench.err
