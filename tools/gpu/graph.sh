timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pytest_gpu.log | grep -E "passed|failed|FAILED|Error" 
timeout 300 python tools/kstats_c2.py 2>&1 | tail -1 | cut -c1-60
PINT_NO_GRAPH=1 timeout 300 python tools/kstats_c2.py 2>&1 | tail -1 | cut -c1-60
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -c 600 gpurun_out/bench.json
