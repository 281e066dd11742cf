set -x
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke.log
timeout 300 python tools/dst_accuracy.py > gpurun_out/dst_acc.json 2>&1; echo "dstacc rc=$?"; cat gpurun_out/dst_acc.json
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_dst_fft|k_band_post2|k_band_pre2|k_band_timeop2|k_band_apply" -c 40 -o gpurun_out/c2_full python tools/kstats_c2.py > gpurun_out/ncu_full.log 2>&1; echo "ncu rc=$?"
tail -3 gpurun_out/ncu_full.log
