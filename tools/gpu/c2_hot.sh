# ncu --set full of the steady-state c2 iteration's hot kernels (tools/prof_c2.py: begin + 1 iteration)
set -x
timeout 900 ncu -f --set full --import-source on --clock-control none -k regex:"k_band_post2" --launch-skip 11 -c 7 -o /tmp/h_post python tools/prof_c2.py 1 > gpurun_out/ncu_h_post.log 2>&1
timeout 900 ncu -f --set full --import-source on --clock-control none -k regex:"k_band_pre2" --launch-skip 9 -c 7 -o /tmp/h_pre python tools/prof_c2.py 1 > gpurun_out/ncu_h_pre.log 2>&1
timeout 900 ncu -f --set full --import-source on --clock-control none -k regex:"k_dst_reg|k_band_timeop2" --launch-skip 1 -c 4 -o /tmp/h_misc python tools/prof_c2.py 1 > gpurun_out/ncu_h_misc.log 2>&1
for r in h_post h_pre h_misc; do
ncu -i /tmp/$r.ncu-rep --page details --csv > gpurun_out/${r}_details.csv 2>&1
ncu -i /tmp/$r.ncu-rep --page source --csv --print-source sass > gpurun_out/${r}_source.csv 2>&1; gzip -f gpurun_out/${r}_source.csv
done
