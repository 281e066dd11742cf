timeout 900 python -m pytest tests/test_gpu_field.py -m gpu -x -q > gpurun_out/pytest_field.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_field.log
timeout 600 python tools/bench_cfg.py --config c4s --steps 3 2>&1 | tail -1
