for spec in "kz_smooth 4" "kz_prolong 4" "kz_z 0" "kz_residual 0"; do
  set -- $spec
  timeout 600 ncu -f --set full --import-source on --clock-control none -k regex:"$1" --launch-skip $2 -c 1 -o /tmp/z_$1 python tools/bench_cfg.py --config c3 --steps 1 > gpurun_out/ncu_$1.log 2>&1
  ncu -i /tmp/z_$1.ncu-rep --page details --csv > gpurun_out/z_$1_details.csv 2>&1
  ncu -i /tmp/z_$1.ncu-rep --page raw --csv > gpurun_out/z_$1_raw.csv 2>&1
  ncu -i /tmp/z_$1.ncu-rep --page source --csv --print-source sass > gpurun_out/z_$1_source.csv 2>&1
done
ls -la gpurun_out | head -30
