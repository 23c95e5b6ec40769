# decode sweep-order A/B on a cfg4 layer (batch 256 x 8K): time + DRAM bytes of the scheduled kernel
for m in 0 1; do
  echo "== KVF_SCHED_HEAD_MINOR=$m"
  KVF_SCHED_HEAD_MINOR=$m python tools/decode_sched_bench.py 1 256 512 2>&1 | tail -5
  KVF_SCHED_HEAD_MINOR=$m timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:"decode_sched_kernel" -c 3 --csv --log-file gpurun_out/dec_ab_$m.csv python tools/decode_sched_bench.py 1 256 512 > /dev/null 2>&1
  python tools/ncu_list.py gpurun_out/dec_ab_$m.csv | tail -3
  grep -h "lts__t_sector_hit_rate" gpurun_out/dec_ab_$m.csv | head -2 | awk -F'","' '{print "L2 hit", $(NF)}'
done
