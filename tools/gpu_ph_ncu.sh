timeout 900 ncu --set full --import-source on --clock-control none -k regex:"sim_tc_kernel" -s 15 -c 3 -o gpurun_out/ph_full python tools/quick_fuse_ph.py 4 > gpurun_out/ph_full.log 2>&1; echo "ncu rc=$?"
ncu -i gpurun_out/ph_full.ncu-rep --page raw --csv > gpurun_out/ph_full_raw.csv 2>/dev/null
ncu -i gpurun_out/ph_full.ncu-rep --page source --csv --launch-skip 2 --launch-count 1 > gpurun_out/ph_full_src.csv 2>/dev/null
