for v in 1 0 1 0 1 0; do KVF_DECODE_SKV=$v timeout 600 python tools/decode_sched_bench.py 1 256 512 > gpurun_out/dec_skv$v.txt 2>&1; echo "skv=$v $(grep fused_sched gpurun_out/dec_skv$v.txt)"; done
