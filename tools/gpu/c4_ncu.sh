# ncu --set full of the field-mode V-cycle kernels on the N=1024 slice of c4
timeout 900 ncu -f --set full --import-source on --clock-control none -k regex:"k_f_smooth|k_f_resid|k_f_x0|k_f_prolong|k_f_restrict|k_f_timeop" --launch-skip 30 -c 24 -o /tmp/c4f python tools/bench_cfg.py --config c4s --steps 1 > gpurun_out/ncu_c4f.log 2>&1
ncu -i /tmp/c4f.ncu-rep --page details --csv > gpurun_out/c4f_details.csv 2>&1
ncu -i /tmp/c4f.ncu-rep --page source --csv --print-source sass > gpurun_out/c4f_source.csv 2>&1; gzip -f gpurun_out/c4f_source.csv
