mkdir -p gpurun_out/r1d
timeout 1200 python bench.py > gpurun_out/r1d/bench.json 2> gpurun_out/r1d/bench.err; tail -2 gpurun_out/r1d/bench.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r1d/bench_ref.json 2>&1; tail -1 gpurun_out/r1d/bench_ref.json | cut -c1-300
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r1d/launches_cfg2.csv python bench.py --steps 1 --warmup 1 --skip-cpu --skip-e2e > /dev/null 2>&1
python tools/ncu_list.py gpurun_out/r1d/launches_cfg2.csv | grep -E "kvf|total|ms "
