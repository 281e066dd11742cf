timeout 900 python bench.py > gpurun_out/bench.jsonl 2> gpurun_out/bench.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref.jsonl 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu > gpurun_out/ncu_launch.log 2>&1; echo "ncu1 rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 700 --csv --log-file gpurun_out/c2_traffic.csv python tools/kstats_c2.py > gpurun_out/c2_traffic.log 2>&1; echo "ncu2 rc=$?"
timeout 600 ncu -f --set full --import-source on --clock-control none -k regex:"k_band_post2|k_dst_reg" -c 3 -o /tmp/c2c python tools/prof_c2.py 1 > gpurun_out/ncu_c2c.log 2>&1; echo "ncu3 rc=$?"
ncu -i /tmp/c2c.ncu-rep --page details --csv > gpurun_out/c2c_details.csv 2>&1
ncu -i /tmp/c2c.ncu-rep --page source --csv --print-source sass > gpurun_out/c2c_source.csv 2>&1; gzip -f gpurun_out/c2c_source.csv
