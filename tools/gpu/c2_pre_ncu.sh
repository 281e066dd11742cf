# ncu --set full of the 2D pre-smoother / coarse band kernels in one steady-state c2 iteration
timeout 900 ncu -f --set full --import-source on --clock-control none -k regex:"k_band_pre2|k_mg_tail" --launch-skip 12 -c 12 -o /tmp/c2pre python tools/prof_c2.py 1 > gpurun_out/ncu_c2pre.log 2>&1
ncu -i /tmp/c2pre.ncu-rep --page details --csv > gpurun_out/c2pre_details.csv 2>&1
ncu -i /tmp/c2pre.ncu-rep --page source --csv --print-source sass > gpurun_out/c2pre_source.csv 2>&1; gzip -f gpurun_out/c2pre_source.csv
