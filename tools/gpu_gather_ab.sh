# compacted levels: staged rows (TMA) vs rows gathered from the pool on the LSU path (cp.async)
timeout 600 python -m pytest tests/test_gpu_tc.py -x -q 2>&1 | tail -2
for cfg in "5 staged" "5 gathered" "4 gathered" "3 gathered" "2 gathered"; do
  set -- $cfg
  timeout 300 python tools/step_breakdown.py 32 64 256 on $1 $2 2>&1 | grep -E "step|similarity_select$|stage_rows$|merge_groups$|Error|error"
done
