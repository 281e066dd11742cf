# round-2 profile set: c2 launch list of the bench command, c3 traffic list,
# ncu --set full of the fused 3D V-cycle kernels
set -x
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/r2_launches.csv python bench.py --steps 2 --warmup 3 --no-other --no-cpu > gpurun_out/r2_launches.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2_c3_traffic.csv python tools/bench_cfg.py --config c3 --steps 1 > gpurun_out/r2_c3_traffic.log 2>&1
bash tools/gpu/c3_ncu.sh
