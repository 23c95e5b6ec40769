# measurement set: GPU suite, smoke, default bench, ncu launch list of one cfg2 fusion step, sim traffic
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.txt 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.txt 2>&1; echo "smoke rc=$?"
timeout 1200 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "bench rc=$?"; head -c 400 gpurun_out/bench_default.json; echo
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_cfg2.csv python bench.py --steps 1 --warmup 0 --skip-cpu --skip-e2e --skip-decode --skip-configs --no-graph > /dev/null 2>&1; echo "ncu list rc=$?"
python tools/ncu_list.py gpurun_out/launches_cfg2.csv | tee gpurun_out/launches_cfg2_summary.txt
bash tools/gpu_sim_traffic.sh
