timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pytest_gpu.log
timeout 300 python tools/dst_accuracy.py 2>&1 | tail -40
timeout 300 python tools/kstats_c2.py 2>&1 | tail -2
PINT_DST_OLD=1 timeout 300 python tools/kstats_c2.py 2>&1 | tail -2
