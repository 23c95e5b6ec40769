# split K / V rings in the sharing-aware decode: tests, then cfg4-layer A/B (interleaved)
timeout 300 python -m pytest tests/test_gpu_decode.py -x -q > gpurun_out/pytest_skv.txt 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_skv.txt
for v in 0 1 0 1; do KVF_DECODE_SKV=$v timeout 600 python tools/decode_sched_bench.py 1 256 512 > gpurun_out/dec_skv$v.txt 2>&1; echo "skv=$v $(grep fused_sched gpurun_out/dec_skv$v.txt)"; done
for v in 0 1; do KVF_DECODE_SKV=$v timeout 600 python tools/decode_cff_bench.py > gpurun_out/dec_cff_skv$v.txt 2>&1; echo "cff skv=$v"; tail -4 gpurun_out/dec_cff_skv$v.txt; done
