# ncu launch list of one cfg2 fusion step (exact mode on / off): time share and DRAM bytes per kernel
for e in on off; do
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"sim_|merge|member|remap|norms|level_stats|state_init|lists_|scales_|rescore|alive_rank|stage_rows|exact|convert|fill|zero" --csv --log-file gpurun_out/launches_exact_$e.csv python bench.py --steps 1 --warmup 1 --skip-cpu --skip-e2e --skip-decode --no-graph --exact $e > /dev/null 2>&1
echo "== exact $e"; python tools/ncu_list.py gpurun_out/launches_exact_$e.csv
done
