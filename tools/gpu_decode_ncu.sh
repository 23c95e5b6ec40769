# ncu --set full of the sharing-aware decode kernel on one cfg4 layer (batch 256 x 8K)
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"decode_sched_kernel" -s 2 -c 1 -o gpurun_out/dec_full python tools/decode_sched_bench.py 1 256 512 > gpurun_out/dec_full.log 2>&1; echo "ncu rc=$?"
ncu -i gpurun_out/dec_full.ncu-rep --page raw --csv > gpurun_out/dec_full_raw.csv 2>/dev/null
ncu -i gpurun_out/dec_full.ncu-rep --page source --csv > gpurun_out/dec_full_src.csv 2>/dev/null
tail -8 gpurun_out/dec_full.log
