timeout 900 python -m pytest tests/test_gpu_minres.py tests/test_gpu_parity.py -m gpu -x -q -s 2>&1 | grep -E "minres|passed|failed|Error|assert" | head -30
