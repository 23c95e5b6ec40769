# cfg1 similarity per level vs the split-K cap
for m in 8 16 4 8 16; do KVF_SPLIT_MAX=$m DTYPE=f32 timeout 600 python tools/step_breakdown.py 4 8 64 > gpurun_out/step_cfg1_s$m.txt 2>&1; echo "max $m"; grep -A8 "^sequence" gpurun_out/step_cfg1_s$m.txt | grep similarity; done
