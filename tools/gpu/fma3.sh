for c in c3 c4s; do
timeout 300 python tools/bench_cfg.py --config $c --steps 3 2>&1 | tail -1 | cut -c1-300
PINT_LIB=$PWD/tools/libpint_fma3.so timeout 300 python tools/bench_cfg.py --config $c --steps 3 2>&1 | tail -1 | cut -c1-300
done
