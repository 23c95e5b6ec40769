timeout 900 ncu --set full --import-source on --clock-control none -k regex:"sim_tc_kernel" -s 12 -c 1 -o gpurun_out/fnorm_l1b python tools/quick_fuse.py 8 > gpurun_out/fnorm_l1b.log 2>&1; echo "ncu rc=$?"
ncu -i gpurun_out/fnorm_l1b.ncu-rep --page raw --csv > gpurun_out/fnorm_l1b_raw.csv 2>/dev/null; ncu -i gpurun_out/fnorm_l1b.ncu-rep --page source --csv > gpurun_out/fnorm_l1b_src.csv 2>/dev/null
KVF_FUSE_KNORM=0 timeout 900 ncu --set full --import-source on --clock-control none -k regex:"sim_tc_kernel" -s 12 -c 1 -o gpurun_out/nofnorm_l1b python tools/quick_fuse.py 8 > gpurun_out/nofnorm_l1b.log 2>&1; echo "ncu rc=$?"
ncu -i gpurun_out/nofnorm_l1b.ncu-rep --page raw --csv > gpurun_out/nofnorm_l1b_raw.csv 2>/dev/null
