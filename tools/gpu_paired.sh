# paired small merges: parity tests, then cfg3 / cfg1 breakdowns paired vs single
timeout 300 python -m pytest tests/test_gpu_paired.py tests/test_gpu_wide.py tests/test_gpu_fused_norms.py -x -q > gpurun_out/pytest_paired.txt 2>&1; echo "pytest rc=$?"; tail -25 gpurun_out/pytest_paired.txt
for pr in 0 1 0 1; do
  KVF_SIM_PAIRED=$pr VARIANT=cff timeout 600 python tools/step_breakdown.py 32 1 1024 > gpurun_out/step_cfg3_p$pr.txt 2>&1; echo "cfg3 paired=$pr rc=$?"; head -4 gpurun_out/step_cfg3_p$pr.txt
  KVF_SIM_PAIRED=$pr DTYPE=f32 timeout 600 python tools/step_breakdown.py 4 8 64 > gpurun_out/step_cfg1_p$pr.txt 2>&1; echo "cfg1 paired=$pr rc=$?"; head -4 gpurun_out/step_cfg1_p$pr.txt
done
