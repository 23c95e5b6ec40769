mkdir -p gpurun_out/merge
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:merge_tma -s 4 -c 2 -o gpurun_out/merge/merge_full python tools/quick_fuse.py 4 > gpurun_out/merge/log 2>&1; tail -2 gpurun_out/merge/log
