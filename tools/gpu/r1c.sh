set -x
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_dst_fft|k_band_post2|k_band_pre2|k_band_timeop2|k_band_apply" -c 40 -o /tmp/c2_full python tools/kstats_c2.py > gpurun_out/ncu_full.log 2>&1; echo "ncu rc=$?"
ncu -i /tmp/c2_full.ncu-rep --page raw --csv > gpurun_out/c2_full_raw.csv 2>&1
ncu -i /tmp/c2_full.ncu-rep --page details --csv > gpurun_out/c2_full_details.csv 2>&1
ls -la /tmp/c2_full.ncu-rep gpurun_out
