timeout 300 python tools/kstats_c2.py 2>&1 | tail -1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_dst_reg" -c 2 -o /tmp/dst python tools/kstats_c2.py > gpurun_out/ncu_dst.log 2>&1; echo "ncu rc=$?"
ncu -i /tmp/dst.ncu-rep --page details --csv > gpurun_out/dst_details.csv 2>&1
ncu -i /tmp/dst.ncu-rep --page raw --csv > gpurun_out/dst_raw.csv 2>&1
ncu -i /tmp/dst.ncu-rep --page source --csv --print-source sass > gpurun_out/dst_source.csv 2>&1
ls -la gpurun_out
