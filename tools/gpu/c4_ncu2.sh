# ncu --set full of the field-mode V-cycle kernels on an N=256 slice of c4 (stored per-step coefficients)
python tools/bench_cfg.py --config c4s --N 256 --steps 1 > gpurun_out/s5_c4s256.json 2>&1 || exit 1
timeout 900 ncu -f --set full --import-source on --clock-control none -k regex:"k_f_smooth|k_f_resid|k_f_x0|k_f_prolong|k_f_restrict|k_f_timeop" --launch-skip 24 -c 26 -o /tmp/c4f python tools/bench_cfg.py --config c4s --N 256 --steps 1 > gpurun_out/ncu_c4f.log 2>&1
ncu -i /tmp/c4f.ncu-rep --page details --csv > gpurun_out/s5_c4f_details.csv 2>&1
