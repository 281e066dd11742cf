timeout 300 python tools/e2e_c2.py 2>&1 | tail -2
PINT_COPY_THREADS=1 timeout 300 python tools/e2e_c2.py 2>&1 | tail -1
nproc; free -g | head -2
