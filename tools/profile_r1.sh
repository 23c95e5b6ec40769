set -x
mkdir -p gpurun_out/prof
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"sim_|merge|member|remap|norms|level_stats|state_init|lists_|scales_|rescore|alive_rank|stage_rows" --csv --log-file gpurun_out/prof/launches_cfg2.csv python bench.py --steps 1 --warmup 1 --skip-cpu --skip-e2e --skip-decode > gpurun_out/prof/bench_under_ncu.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sim_tc_kernel -s 6 -c 6 -o gpurun_out/prof/sim_tc python tools/quick_fuse.py 4 > gpurun_out/prof/ncu_sim.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:merge_kernel -s 6 -c 6 -o gpurun_out/prof/merge python tools/quick_fuse.py 4 > gpurun_out/prof/ncu_merge.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"decode_fast|block_norms" -s 2 -c 3 -o gpurun_out/prof/decode python tools/decode_only.py > gpurun_out/prof/ncu_decode.log 2>&1
ls -la gpurun_out/prof
