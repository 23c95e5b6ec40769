# per-rank work at 8 GPUs (4 layers of cfg2): wide auto vs narrow, per-level similarity times
for w in auto 0 auto 0; do KVF_SIM_WIDE=$w timeout 600 python tools/step_breakdown.py 4 > gpurun_out/step_u4_$w.txt 2>&1; echo "wide=$w $(head -1 gpurun_out/step_u4_$w.txt | cut -c1-120)"; grep "^level [1-6]: sim" gpurun_out/step_u4_$w.txt | cut -c1-40; done
