PINT_ARITH=exact timeout 300 python tools/c2_history.py > gpurun_out/h_exact.json 2>&1
PINT_ARITH=fast timeout 300 python tools/c2_history.py > gpurun_out/h_fast.json 2>&1
PINT_ARITH=exact PINT_AREF_SEPARATE=1 timeout 300 python tools/c2_history.py > gpurun_out/h_exact_sep.json 2>&1
PINT_ARITH=fast PINT_AREF_SEPARATE=1 timeout 300 python tools/c2_history.py > gpurun_out/h_fast_sep.json 2>&1
