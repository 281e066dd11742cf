timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
timeout 300 python tools/kstats_c2.py 2>&1 | tail -1
timeout 300 python tools/kstats_c2.py 2>&1 | tail -1
