# ncu --set full of the wide similarity tile (4-layer cfg2 shape, levels 3-6)
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"sim_tc_kernel" -s 14 -c 6 -o gpurun_out/sim4w_full python tools/quick_fuse.py 4 > gpurun_out/sim4w_full.log 2>&1; echo "sim rc=$?"
ncu -i gpurun_out/sim4w_full.ncu-rep --page raw --csv > gpurun_out/sim4w_full_raw.csv 2>/dev/null
tail -3 gpurun_out/sim4w_full.log
