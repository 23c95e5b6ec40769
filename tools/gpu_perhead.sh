# per-head units (north star granularity): cfg2 per-call breakdown, wide forced vs auto
HEAD_MODE=1 timeout 900 python tools/step_breakdown.py > gpurun_out/step_cfg2_perhead.txt 2>&1; echo "perhead rc=$?"; head -60 gpurun_out/step_cfg2_perhead.txt
HEAD_MODE=1 KVF_SIM_WIDE=1 timeout 900 python tools/step_breakdown.py > gpurun_out/step_cfg2_perhead_wide.txt 2>&1; echo "perhead wide rc=$?"; head -12 gpurun_out/step_cfg2_perhead_wide.txt
