# after the wide tile: GPU suite, default bench, ncu traffic of one cfg2 step's similarity launches
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.txt 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.txt
timeout 1200 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "bench rc=$?"
head -c 1500 gpurun_out/bench_default.json
bash tools/gpu_sim_traffic.sh
