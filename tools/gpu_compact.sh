timeout 600 python -m pytest tests/test_compact.py tests/test_gpu_decode.py -x -q 2>&1 | tail -2
timeout 1200 python bench.py --steps 3 --warmup 3 --skip-cpu --skip-e2e 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(json.dumps(d['decode'], indent=1))"
