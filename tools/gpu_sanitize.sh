# compute-sanitizer over tools/sanitize_small.py: memcheck, synccheck, initcheck, racecheck
# (racecheck in analysis mode: one line per distinct hazard; the summary is classified in
# profiles/r02_sanitizer.md)
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck synccheck initcheck; do
  timeout 1200 $CS --tool $tool --print-limit 200 python tools/sanitize_small.py > gpurun_out/san_$tool.txt 2>&1
  echo "== $tool rc=$?"; tail -4 gpurun_out/san_$tool.txt
done
timeout 1800 $CS --tool racecheck --racecheck-report analysis --print-limit 100000 python tools/sanitize_small.py > gpurun_out/san_racecheck.txt 2>&1
echo "== racecheck rc=$?"; tail -4 gpurun_out/san_racecheck.txt
