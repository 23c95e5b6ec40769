# decode item size A/B on a cfg4 layer: time + DRAM bytes of the scheduled kernel
for ib in 16 8; do
  echo "== IB=$ib"
  IB=$ib python tools/decode_sched_bench.py 1 256 512 2>&1 | grep -E "fused_sched|IB="
  IB=$ib timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"decode_sched_kernel|combine" -c 6 --csv --log-file gpurun_out/dec_ib_$ib.csv python tools/decode_sched_bench.py 1 256 512 > /dev/null 2>&1
  python tools/ncu_list.py gpurun_out/dec_ib_$ib.csv | tail -4
done
