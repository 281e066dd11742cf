# device diagnostics + parity reruns
timeout 1200 python -m pytest tests/test_gpu_diagnostics.py tests/test_gpu_3d.py tests/test_gpu_minres.py tests/test_gpu_table2.py tests/test_problem_io.py tests/test_gpu_parity.py -m gpu -q -rs > gpurun_out/pytest_b.log 2>&1; echo "pytest rc=$?"; grep -E "passed|failed|FAILED|Error|drift|floor" gpurun_out/pytest_b.log | tail -30
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
