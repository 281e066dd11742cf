timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "dst or DST or htilde or uzawa or config1" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
for pf in 0 1; do PINT_DST_PF=$pf timeout 300 python tools/kstats_c2.py 2>&1 | tail -1; done
