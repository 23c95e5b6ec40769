mkdir -p gpurun_out/mab
for cfg in "148 204800" "296 102400" "296 98304" "444 65536"; do set -- $cfg
KVF_MERGE_CTAS=$1 KVF_MERGE_SMEM=$2 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:merge_tma --csv --log-file gpurun_out/mab/m_$1_$2.csv python tools/quick_fuse.py 4 > /dev/null 2>&1
echo "ctas $1 smem $2"; python tools/ncu_list.py gpurun_out/mab/m_$1_$2.csv | grep merge
done
