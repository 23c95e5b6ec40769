# One `ncu --set full` capture of the similarity kernel over one eager cfg2 fusion step
# -> profiles/cfg2_sim_traffic.json (DRAM bytes per launch, the bench's roofline.traffic)
# and a raw-page CSV of the launches for reading here.
timeout 2400 ncu --set full --import-source on --clock-control none -k regex:"sim_tc_kernel" -c 12 \
  -o gpurun_out/sim_full python bench.py --steps 1 --warmup 0 --skip-cpu --skip-e2e --skip-decode \
  --skip-configs --no-graph > gpurun_out/sim_full.log 2>&1
echo "ncu rc=$?"
ncu -i gpurun_out/sim_full.ncu-rep --page raw --csv > gpurun_out/sim_full_raw.csv 2>/dev/null
python - <<'PY'
import csv, json, subprocess
rows = list(csv.reader(open("gpurun_out/sim_full_raw.csv")))
h = rows[0]
units = rows[1]
data = rows[2:]
def col(name):
    return h.index(name)
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}
rd, wr, t = col("dram__bytes_read.sum"), col("dram__bytes_write.sum"), col("gpu__time_duration.sum")
tot, per = 0.0, []
for r in data:
    b = float(r[rd].replace(",", "")) * scale.get(units[rd], 1) + float(r[wr].replace(",", "")) * scale.get(units[wr], 1)
    per.append(b)
    tot += b
tensor = [c for c in h if "pipe_tensor" in c and "pct" in c]
head = subprocess.run(["git", "rev-parse", "--short", "HEAD"], capture_output=True, text=True).stdout.strip()
out = {"kernel": "sim_tc_kernel", "launches": len(per), "bytes_per_launch": tot / max(1, len(per)),
       "bytes_per_step": tot, "per_launch_bytes": per, "source": "ncu --set full --clock-control none, "
       "one eager cfg2 fusion step (bench.py --steps 1 --warmup 0 --no-graph)", "head": head}
json.dump(out, open("profiles/cfg2_sim_traffic.json", "w"), indent=1)
print(json.dumps({k: v for k, v in out.items() if k != "per_launch_bytes"}))
PY
