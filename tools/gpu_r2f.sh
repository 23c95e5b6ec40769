# full GPU suite (no -x) + warm per-launch breakdown of one cfg2 step
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.txt 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pytest_gpu.txt
timeout 600 python tools/step_breakdown.py > gpurun_out/step_cfg2.txt 2>&1; echo "breakdown rc=$?"; head -40 gpurun_out/step_cfg2.txt
