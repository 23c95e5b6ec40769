set -x
mkdir -p gpurun_out/r1b
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/r1b/pytest_gpu.log 2>&1; tail -3 gpurun_out/r1b/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r1b/smoke.log 2>&1; tail -2 gpurun_out/r1b/smoke.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/r1b/bench.json 2> gpurun_out/r1b/bench.err; tail -3 gpurun_out/r1b/bench.err; cat gpurun_out/r1b/bench.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r1b/launches_cfg2.csv python bench.py --steps 1 --warmup 1 --skip-cpu --skip-e2e --skip-decode > gpurun_out/r1b/bench_under_ncu.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sim_tc_kernel -s 6 -c 6 -o gpurun_out/r1b/sim_tc python tools/quick_fuse.py 4 > gpurun_out/r1b/ncu_sim.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:merge_kernel -s 6 -c 6 -o gpurun_out/r1b/merge python tools/quick_fuse.py 4 > gpurun_out/r1b/ncu_merge.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"decode|block_norms" -s 2 -c 4 -o gpurun_out/r1b/decode python tools/decode_only.py > gpurun_out/r1b/ncu_decode.log 2>&1
ls -la gpurun_out/r1b
