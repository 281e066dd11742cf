# fused 3D band V-cycle: parity + A/B timing
timeout 900 python -m pytest tests/test_gpu_3d.py tests/test_gpu_diagnostics.py -m gpu -q -x > gpurun_out/pytest_c.log 2>&1; echo "pytest rc=$?"; grep -E "passed|failed|FAILED|Error|drift|floor" gpurun_out/pytest_c.log | tail -20
for v in "" "PINT_3D_OLD=1"; do env $v timeout 600 python tools/bench_cfg.py --config c3 --steps 3 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', d['ms_per_iter'], {k:round(v['ms'],3) for k,v in d['kernels'].items()})"; done
