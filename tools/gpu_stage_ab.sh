# staging budget A/B (interleaved): 4 GB = 4 unit chunks of 8 layers, 24 GB = one chunk
for b in 4 24 4 24; do KVF_STAGE_BUDGET=$b timeout 600 python tools/step_breakdown.py > gpurun_out/step_cfg2_stage_$b.txt 2>&1; echo "budget $b rc=$?"; head -3 gpurun_out/step_cfg2_stage_$b.txt; done
