# chunked level statistics: parity tests, GPU suite, cfg5 layer + cfg2 step breakdowns
timeout 900 python -m pytest tests/test_gpu_level_stats.py -x -q > gpurun_out/pytest_ls.txt 2>&1; echo "pytest ls rc=$?"; tail -15 gpurun_out/pytest_ls.txt
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.txt 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.txt
timeout 900 python tools/step_breakdown.py 1 256 1024 > gpurun_out/step_cfg5_ls.txt 2>&1; echo "cfg5 rc=$?"; head -12 gpurun_out/step_cfg5_ls.txt
timeout 600 python tools/step_breakdown.py > gpurun_out/step_cfg2_ls.txt 2>&1; echo "cfg2 rc=$?"; head -12 gpurun_out/step_cfg2_ls.txt
