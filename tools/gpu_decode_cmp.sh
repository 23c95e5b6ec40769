timeout 300 python -m pytest tests/test_gpu_decode.py -q -x 2>&1 | tail -1
for c in 0 1 2 3; do KVF_DECODE_CFG=$c python tools/decode_bench.py; done
