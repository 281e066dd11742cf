for h in 4 2; do PINT_AR_HC=$h timeout 300 python tools/kstats_c2.py 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['env'], d['ms_per_step'], {k:v for k,v in d['ms'].items() if 'fine' in k})"; done
PINT_AR_HC=2 timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "fused or band" 2>&1 | tail -1
