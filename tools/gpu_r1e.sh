mkdir -p gpurun_out/r1e
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sim_tc_kernel -c 6 -o gpurun_out/r1e/sim_tc python tools/quick_fuse.py 4 > gpurun_out/r1e/ncu_sim.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:merge_tma -c 6 -o gpurun_out/r1e/merge python tools/quick_fuse.py 4 > gpurun_out/r1e/ncu_merge.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:decode_sched -c 2 -o gpurun_out/r1e/decode_sched python tools/decode_sched_bench.py 1 64 256 > gpurun_out/r1e/ncu_dec.log 2>&1
ls gpurun_out/r1e
