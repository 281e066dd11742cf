timeout 300 python tools/kstats_c2.py 2>&1 | tail -1
PINT_DST_MINB=1 timeout 300 python tools/kstats_c2.py 2>&1 | tail -1
PINT_DST_P=2 timeout 300 python tools/kstats_c2.py 2>&1 | tail -1
PINT_DST_P=2 PINT_DST_MINB=1 timeout 300 python tools/kstats_c2.py 2>&1 | tail -1
