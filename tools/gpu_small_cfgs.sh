# per-call breakdowns of cfg3 (CFF 8 x 2K, 32 layers) and cfg1 (fp32, 4 layers) fusion steps
VARIANT=cff timeout 600 python tools/step_breakdown.py 32 1 1024 > gpurun_out/step_cfg3.txt 2>&1; echo "cfg3 rc=$?"; cat gpurun_out/step_cfg3.txt | head -60
DTYPE=f32 timeout 600 python tools/step_breakdown.py 4 8 64 > gpurun_out/step_cfg1.txt 2>&1; echo "cfg1 rc=$?"; cat gpurun_out/step_cfg1.txt | head -60
