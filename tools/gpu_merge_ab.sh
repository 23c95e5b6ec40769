# merge kernel A/B: dynamic item fetch + ring-fed shadow rows; ring depth
timeout 900 python -m pytest tests/test_gpu_exact.py tests/test_gpu_parity.py tests/test_gpu_determinism.py tests/test_gpu_golden.py -x -q 2>&1 | tail -2
for nb in 2 3; do echo "== nbuf $nb"; KVF_MERGE_NBUF=$nb python tools/step_breakdown.py 32 64 256 on 2>&1 | grep -E "step|merge_groups$|level [0-9]"; done
python tools/step_breakdown.py 32 64 256 off 2>&1 | grep -E "step|merge_groups$|level [0-9]"
