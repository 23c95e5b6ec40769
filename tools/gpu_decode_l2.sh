# sharing-aware decode: L2 eviction policy A/B (KVF_DECODE_L2 = 0 none, 1 evict-first for
# single-reference blocks, 2 + evict-last for shared blocks) on a cfg4 layer
timeout 600 python -m pytest tests/test_gpu_decode.py -x -q 2>&1 | tail -2
for m in 0 1 2; do echo "== KVF_DECODE_L2=$m"; KVF_DECODE_L2=$m python tools/decode_sched_bench.py 2 256 512 2>&1 | grep -E "fused_sched|CR"; done
KVF_DECODE_L2=1 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:decode_sched_kernel -s 3 -c 1 python tools/decode_sched_bench.py 1 256 512 2>&1 | grep -E "duration|bytes|hit_rate"
KVF_DECODE_L2=0 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:decode_sched_kernel -s 3 -c 1 python tools/decode_sched_bench.py 1 256 512 2>&1 | grep -E "duration|bytes|hit_rate"
