set -x
mkdir -p gpurun_out/sched
timeout 600 python -m pytest tests/test_gpu_decode.py -x -q > gpurun_out/sched/pytest.log 2>&1; tail -15 gpurun_out/sched/pytest.log
IB=16 timeout 600 python tools/decode_sched_bench.py 2 64 256 2>&1 | tail -8
IB=8 timeout 600 python tools/decode_sched_bench.py 2 64 256 2>&1 | tail -8
IB=16 timeout 900 python tools/decode_sched_bench.py 4 256 512 2>&1 | tail -8
IB=16 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:"decode_" --csv --log-file gpurun_out/sched/ncu_decode.csv python tools/decode_sched_bench.py 1 64 256 > /dev/null 2>&1
python tools/ncu_list.py gpurun_out/sched/ncu_decode.csv 2>&1 | head
IB=16 timeout 600 ncu --set full --import-source on --clock-control none -k regex:"decode_sched" -c 2 -o gpurun_out/sched/sched_full python tools/decode_sched_bench.py 1 64 256 > /dev/null 2>&1
ls gpurun_out/sched
