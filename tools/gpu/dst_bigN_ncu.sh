# DRAM traffic of the sine transforms at N = 4096 / 8192 (2- and 4-column tiles): ncu launch list with dram bytes
for N in 4096 8192; do
python tools/gpu/dst_bigN.py $N 256 > gpurun_out/s5_dst_bigN_$N.log 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:k_dst -c 6 --csv --log-file gpurun_out/s5_dst_bigN_${N}_ncu.csv python tools/gpu/dst_bigN.py $N 256 > /dev/null 2>&1
done
cat gpurun_out/s5_dst_bigN_*.log
