timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"sim_|merge|member|remap|norms|level_stats|state_init|lists_|scales_" --csv --log-file gpurun_out/launches_q.csv python tools/quick_fuse.py 4 > /dev/null 2>&1
python tools/ncu_list.py gpurun_out/launches_q.csv
python -m pytest tests/test_gpu_tc.py -x -q 2>&1 | grep -E "^E" | head -5
