# wide similarity tile: parity tests, then cfg2 step breakdown wide (auto) vs narrow
timeout 900 python -m pytest tests/test_gpu_wide.py tests/test_gpu_tc.py tests/test_gpu_splitk.py -x -q > gpurun_out/pytest_wide.txt 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pytest_wide.txt
for w in auto 0 auto; do
  KVF_SIM_WIDE=$w timeout 600 python tools/step_breakdown.py > gpurun_out/step_cfg2_wide_$w.txt 2>&1; echo "breakdown $w rc=$?"; head -12 gpurun_out/step_cfg2_wide_$w.txt
done
