# bench.py CLI paths besides the default line
for a in "--config cfg1" "--config cfg3" "--head-mode per_head" "--exact off"; do
  timeout 900 python bench.py $a --skip-cpu --skip-e2e --skip-decode --skip-configs --steps 3 --warmup 3 > gpurun_out/cli.json 2> gpurun_out/cli.err; rc=$?
  python -c "
import json,sys
d=json.load(open('gpurun_out/cli.json')); print('$a', 'rc=$rc', round(d['ms_per_step'],3), 'ms', round(d['value'],1), d['unit'], 'CR', round(d['compression_ratio'],4), 'frac', round(d['roofline']['frac'] or 0,3))" 2>&1 | tail -1
done
