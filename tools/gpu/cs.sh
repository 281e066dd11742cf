for lib in "" "$PWD/tools/libpint_cs.so"; do PINT_LIB=$lib timeout 300 python tools/bench_cfg.py --config c3 --steps 3 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_iter'], {k:v['ms'] for k,v in d['kernels'].items()})"; done
PINT_LIB=$PWD/tools/libpint_cs.so timeout 600 python -m pytest tests/test_gpu_3d.py -m gpu -q 2>&1 | tail -1
