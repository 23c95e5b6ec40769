# sharing-aware decode: L2 prefetch distance A/B on a cfg4 layer (batch 256 x 8K)
for pf in 0 2 4 8 0 3 6; do KVF_DECODE_PF=$pf timeout 600 python tools/decode_sched_bench.py 1 256 512 > gpurun_out/dec_pf$pf.txt 2>&1; echo "pf=$pf $(grep fused_sched gpurun_out/dec_pf$pf.txt)"; done
