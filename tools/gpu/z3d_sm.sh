timeout 600 ncu -f --set full --import-source on --clock-control none -k regex:"kz_smooth" --launch-skip 4 -c 1 -o /tmp/z_sm python tools/bench_cfg.py --config c3 --steps 1 > gpurun_out/ncu_zsm.log 2>&1; echo rc=$?
ncu -i /tmp/z_sm.ncu-rep --page details --csv > gpurun_out/z_sm_details.csv 2>&1
ncu -i /tmp/z_sm.ncu-rep --page source --csv --print-source sass > gpurun_out/z_sm_source.csv 2>&1; gzip -f gpurun_out/z_sm_source.csv
