# A/B of the similarity tile launch order (KVF_TILE_BAND) on cfg2: step time and the
# similarity kernel's DRAM bytes per level (ncu, one eager step)
for b in ${BANDS:-4 8 12}; do
  KVF_TILE_BAND=$b python bench.py --steps 10 --warmup 3 --skip-cpu --skip-e2e --skip-decode --skip-configs > gpurun_out/band_$b.json 2>&1
  python -c "import json;d=json.load(open('gpurun_out/band_$b.json'));print('band $b', round(d['ms_per_step'],2), round(d['roofline']['achieved']), d['clocks']['sm_mhz'])"
  KVF_TILE_BAND=$b timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"sim_tc" --csv --log-file gpurun_out/band_$b.csv python bench.py --steps 1 --warmup 0 --skip-cpu --skip-e2e --skip-decode --skip-configs --no-graph > /dev/null 2>&1
  python - <<PY
import csv
rows=list(csv.reader(open("gpurun_out/band_$b.csv")))
h=next(i for i,r in enumerate(rows) if r and r[0]=="ID"); H=rows[h]
ni,vi,ui=H.index("Metric Name"),H.index("Metric Value"),H.index("Metric Unit")
t=[];rd=[]
for r in rows[h+1:]:
    v=float(r[vi].replace(",",""))
    if r[ni]=="gpu__time_duration.sum": t.append(v*(1e-3 if r[ui] in("us","usecond") else 1e-6 if r[ui] in("ns","nsecond") else 1))
    if r[ni]=="dram__bytes_read.sum": rd.append(v*{"byte":1e-9,"Kbyte":1e-6,"Mbyte":1e-3,"Gbyte":1}[r[ui]])
print("band $b per level ms", [round(x,2) for x in t[-6:]], "read GB", [round(x,2) for x in rd[-6:]])
PY
done
