# ncu --set full of the top-level merge launches (4-layer cfg2 shape, third run)
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"merge_tma_kernel" -s 14 -c 4 -o gpurun_out/merge4_full python tools/quick_fuse.py 4 > gpurun_out/merge4_full.log 2>&1; echo "ncu rc=$?"
ncu -i gpurun_out/merge4_full.ncu-rep --page raw --csv > gpurun_out/merge4_full_raw.csv 2>/dev/null
ncu -i gpurun_out/merge4_full.ncu-rep --page details --csv > gpurun_out/merge4_full_details.csv 2>/dev/null
tail -2 gpurun_out/merge4_full.log
