# ncu --set full of the sine transforms: cluster kernel at N = 4096, single-CTA kernels at N = 4096 and N = 1024
ncu -f --set full --clock-control none -k regex:k_dst --launch-skip 2 -c 2 -o /tmp/dcl python tools/gpu/dst_bigN.py 4096 256 > gpurun_out/ncu_dcl.log 2>&1
ncu -i /tmp/dcl.ncu-rep --page details --csv > gpurun_out/s5_dcl_details.csv 2>&1
PINT_DST_NOCL=1 ncu -f --set full --clock-control none -k regex:k_dst --launch-skip 2 -c 2 -o /tmp/dnc python tools/gpu/dst_bigN.py 4096 256 > gpurun_out/ncu_dnc.log 2>&1
ncu -i /tmp/dnc.ncu-rep --page details --csv > gpurun_out/s5_dnc_details.csv 2>&1
ncu -f --set full --clock-control none -k regex:k_dst --launch-skip 2 -c 2 -o /tmp/d1k python tools/gpu/dst_bigN.py 1024 256 > gpurun_out/ncu_d1k.log 2>&1
ncu -i /tmp/d1k.ncu-rep --page details --csv > gpurun_out/s5_d1k_details.csv 2>&1
