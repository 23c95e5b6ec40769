# ncu --set full: cuBLAS bf16 8192^3 vs sim_tc_kernel (4-layer cfg2 shape, levels 3-6)
timeout 600 ncu --set full --clock-control none -k regex:"nvjet|gemm|sm100" -s 10 -c 2 -o gpurun_out/mm_full python tools/mm_probe.py > gpurun_out/mm_full.log 2>&1; echo "mm rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"sim_tc_kernel" -s 14 -c 6 -o gpurun_out/sim4_full python tools/quick_fuse.py 4 > gpurun_out/sim4_full.log 2>&1; echo "sim rc=$?"
for f in mm_full sim4_full; do ncu -i gpurun_out/$f.ncu-rep --page raw --csv > gpurun_out/${f}_raw.csv 2>/dev/null; done
ls -la gpurun_out
