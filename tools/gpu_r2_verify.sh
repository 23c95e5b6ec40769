# full GPU suite + sanitizers after the merge / gather changes
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu2.txt 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu2.txt
bash tools/gpu_sanitize.sh
