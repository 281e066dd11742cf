timeout 900 python -m pytest tests/test_gpu_3d.py -m gpu -x -q > gpurun_out/pytest_3d.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_3d.log
timeout 300 python tools/bench_cfg.py --config c3 2>&1 | tail -1
