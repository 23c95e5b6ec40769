for v in 0 1 2; do KVF_SCHED_VARIANT=$v IB=16 timeout 600 python tools/decode_sched_bench.py 2 64 256 2>&1 | grep "sched "; done
for v in 1 2; do KVF_SCHED_VARIANT=$v timeout 600 python -m pytest tests/test_gpu_decode.py -x -q 2>&1 | tail -1; done
