timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pytest_gpu.log | grep -E "passed|failed|FAILED|Error" 
PINT_ARITH=exact timeout 300 python tools/c2_history.py > gpurun_out/h_exact.json 2>&1
PINT_ARITH=fast timeout 300 python tools/c2_history.py > gpurun_out/h_fast.json 2>&1
timeout 300 python tools/kstats_c2.py 2>&1 | tail -1 | cut -c1-60
