timeout 300 python tools/kstats_c2.py 2>&1 | tail -1
PINT_LIB=$PWD/tools/libpint_fma.so timeout 300 python tools/kstats_c2.py 2>&1 | tail -1
