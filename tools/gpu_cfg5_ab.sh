# cfg5 layer (262,144 blocks): per-call breakdown, wide auto vs narrow
for w in auto 0; do
  KVF_SIM_WIDE=$w timeout 900 python tools/step_breakdown.py 1 256 1024 > gpurun_out/step_cfg5_wide_$w.txt 2>&1; echo "cfg5 $w rc=$?"; head -12 gpurun_out/step_cfg5_wide_$w.txt
done
