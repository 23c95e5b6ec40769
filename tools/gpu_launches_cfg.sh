# ncu launch list (kvf kernels) of one fusion step for a config, split-K on / off:
#   bash tools/gpu_launches_cfg.sh cfg1
c=${1:-cfg1}
for sp in "" "--no-split"; do
tag=${sp:-split}; tag=${tag#--}
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"kvf::|sim_|merge|norms|rescore|convert|level_stats|remap" --csv --log-file gpurun_out/launches_${c}_${tag}.csv python bench.py --config $c --steps 1 --warmup 1 --skip-cpu --skip-e2e --skip-decode --no-graph $sp > /dev/null 2>&1
echo "== $c $tag"; python tools/ncu_list.py gpurun_out/launches_${c}_${tag}.csv
done
