timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pytest_gpu.log | grep -E "passed|failed|FAILED|Error"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
