# ncu of the level-1 similarity launch with fused key norms (4-layer cfg2 shape, third run)
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"sim_tc_kernel" -s 12 -c 1 -o gpurun_out/fnorm_l1 python tools/quick_fuse.py 4 > gpurun_out/fnorm_l1.log 2>&1; echo "ncu rc=$?"
KVF_FUSE_KNORM=0 timeout 900 ncu --set full --import-source on --clock-control none -k regex:"sim_tc_kernel" -s 12 -c 1 -o gpurun_out/nofnorm_l1 python tools/quick_fuse.py 4 > gpurun_out/nofnorm_l1.log 2>&1; echo "ncu rc=$?"
for f in fnorm_l1 nofnorm_l1; do ncu -i gpurun_out/$f.ncu-rep --page raw --csv > gpurun_out/${f}_raw.csv 2>/dev/null; ncu -i gpurun_out/$f.ncu-rep --page source --csv > gpurun_out/${f}_src.csv 2>/dev/null; done
ls -la gpurun_out/*_l1*
