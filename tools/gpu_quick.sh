python -m pytest tests -x -q -m gpu 2>&1 | tail -5
timeout 300 python tools/quick_fuse.py 32 2>&1 | tail -4
