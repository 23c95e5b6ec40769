timeout 600 python -m pytest tests/test_gpu_tc.py -x -q 2>&1 | tail -2
timeout 600 python bench.py --steps 5 --warmup 3 --skip-cpu --skip-e2e --skip-decode 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['ms_per_step'], d['value'], d['roofline']['sim_ms_per_step'])"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"stage_rows|gather_rows|merge|norms" --csv --log-file gpurun_out/stage.csv python bench.py --steps 1 --warmup 1 --skip-cpu --skip-e2e --skip-decode > /dev/null 2>&1
python tools/ncu_list.py gpurun_out/stage.csv
