# ncu --set full of the fused 3D V-cycle kernels on c3 (begin + 1 iteration):
# V-cycles 4-6 are the iteration's (A~ with the p update, H~ first, H~ second)
set -x
timeout 900 ncu -f --set full --import-source on --clock-control none -k regex:kc3_post --launch-skip 19 -c 11 -o /tmp/c3_post python tools/bench_cfg.py --config c3 --steps 1 > gpurun_out/ncu_c3_post.log 2>&1
timeout 900 ncu -f --set full --import-source on --clock-control none -k regex:kc3_pre --launch-skip 15 -c 11 -o /tmp/c3_pre python tools/bench_cfg.py --config c3 --steps 1 > gpurun_out/ncu_c3_pre.log 2>&1
for r in c3_post c3_pre; do
ncu -i /tmp/$r.ncu-rep --page details --csv > gpurun_out/${r}_details.csv 2>&1
ncu -i /tmp/$r.ncu-rep --page source --csv --print-source sass > gpurun_out/${r}_source.csv 2>&1; gzip -f gpurun_out/${r}_source.csv
done
