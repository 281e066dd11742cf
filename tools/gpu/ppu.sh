timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pytest_gpu.log | grep -E "passed|failed|FAILED|Error" 
for k in 0 1; do PINT_PPU=$k timeout 300 python tools/kstats_c2.py 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['env'], d['ms_per_step'], {k:v for k,v in d['ms'].items() if 'mg' in k})"; done
timeout 300 python tools/c2_history.py > gpurun_out/h_fast.json 2>&1
