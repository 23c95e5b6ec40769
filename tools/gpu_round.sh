set -x
python -m pytest tests -x -q -m gpu 2>&1 | tail -5
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_r1a.json 2> gpurun_out/bench_r1a.err; tail -3 gpurun_out/bench_r1a.err
cat gpurun_out/bench_r1a.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"sim_|merge_|remap|norms|level_stats|state_init|lists_|scales_" --csv --log-file gpurun_out/launches_r1.csv python bench.py --steps 1 --warmup 1 --skip-cpu --skip-e2e --skip-decode > /dev/null 2>&1; wc -l gpurun_out/launches_r1.csv
