mkdir -p gpurun_out/r1c
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
timeout 900 python bench.py --head-mode per_head --steps 5 --warmup 3 --skip-cpu --skip-e2e --skip-decode > gpurun_out/r1c/bench_perhead.json 2> gpurun_out/r1c/bench_perhead.err; tail -2 gpurun_out/r1c/bench_perhead.err
python -c "import json; d=json.load(open('gpurun_out/r1c/bench_perhead.json')); print(d['ms_per_step'], d['value'], d['compression_ratio'], d['roofline']['frac'], d['roofline']['sim_ms_per_step'])"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"merge|sim_tc" --csv --log-file gpurun_out/r1c/launches_perhead.csv python bench.py --head-mode per_head --steps 1 --warmup 1 --skip-cpu --skip-e2e --skip-decode > /dev/null 2>&1
python tools/ncu_list.py gpurun_out/r1c/launches_perhead.csv | grep -E "kvf|total"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:sim_tc -s 4 -c 1 -o gpurun_out/r1c/sim_perhead python bench.py --head-mode per_head --steps 1 --warmup 0 --skip-cpu --skip-e2e --skip-decode > /dev/null 2>&1; ls gpurun_out/r1c
