# ncu --set full of the c2 hot kernels (DST pair, fine pre-smoother, r1/z time operators)
set -x
timeout 600 ncu -f --set full --import-source on --clock-control none -k regex:"k_dst_reg|k_band_timeop2" -c 4 -o /tmp/c2a python tools/prof_c2.py 1 > gpurun_out/ncu_c2a.log 2>&1; echo "ncu rc=$?"
timeout 600 ncu -f --set full --import-source on --clock-control none -k regex:"k_band_pre2|k_band_post2" -c 2 -o /tmp/c2b python tools/prof_c2.py 1 > gpurun_out/ncu_c2b.log 2>&1; echo "ncu rc=$?"
for r in c2a c2b; do
ncu -i /tmp/$r.ncu-rep --page details --csv > gpurun_out/${r}_details.csv 2>&1
ncu -i /tmp/$r.ncu-rep --page source --csv --print-source sass > gpurun_out/${r}_source.csv 2>&1
gzip -f gpurun_out/${r}_source.csv
done
