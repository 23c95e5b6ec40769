timeout 300 python -m pytest tests/test_gpu_fused_norms.py tests/test_gpu_paired.py -x -q > gpurun_out/pytest_dec.txt 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pytest_dec.txt
timeout 600 python -m pytest tests/test_gpu_exact.py tests/test_gpu_parity.py tests/test_gpu_golden.py tests/test_gpu_determinism.py -x -q > gpurun_out/pytest_dec2.txt 2>&1; echo "pytest2 rc=$?"; tail -3 gpurun_out/pytest_dec2.txt
for v in base new base new; do
  if [ "$v" = base ]; then LIB=_ab/base.so; else LIB=paper_2601_03067_b200/_lib/libkvfuse_b200.so; fi
  KVF_LIB=$LIB timeout 600 python tools/step_breakdown.py > gpurun_out/ab_$v.txt 2>&1
  echo "$v: $(head -1 gpurun_out/ab_$v.txt | sed 's/.*step/step/') L1 $(grep -A3 '^sequence' gpurun_out/ab_$v.txt | grep similarity | head -1)"
done
