for v in 0 1 2 3 0; do KVF_SCHED_VARIANT=$v IB=16 timeout 600 python tools/decode_sched_bench.py 2 64 256 2>&1 | grep "sched "; done
