# round-1 v8: bench line, launch list of the bench command, hot-kernel ncu captures, DRAM traffic list
set -x
mkdir -p gpurun_out
python bench.py > gpurun_out/v8_bench.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/v8_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-other > gpurun_out/v8_launches.log 2>&1
bash tools/gpu/c2_hot.sh
