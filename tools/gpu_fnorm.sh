# fused level-1 key norms: parity tests, cfg2 breakdown A/B (level-1 launch times), ncu of the launch
timeout 300 python -m pytest tests/test_gpu_fused_norms.py -x -q > gpurun_out/pytest_fnorm.txt 2>&1; echo "pytest fnorm rc=$?"; tail -3 gpurun_out/pytest_fnorm.txt
for f in 0 1 0 1; do KVF_FUSE_KNORM=$f timeout 600 python tools/step_breakdown.py > gpurun_out/step_cfg2_fnorm_$f.txt 2>&1; echo "fnorm $f rc=$?"; head -1 gpurun_out/step_cfg2_fnorm_$f.txt; grep -A4 "^sequence" gpurun_out/step_cfg2_fnorm_$f.txt; done
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"sim_tc_kernel" -s 12 -c 1 -o gpurun_out/fnorm_l1 python tools/quick_fuse.py 4 > gpurun_out/fnorm_l1.log 2>&1; echo "ncu rc=$?"
ncu -i gpurun_out/fnorm_l1.ncu-rep --page raw --csv > gpurun_out/fnorm_l1_raw.csv 2>/dev/null; ncu -i gpurun_out/fnorm_l1.ncu-rep --page source --csv > gpurun_out/fnorm_l1_src.csv 2>/dev/null
