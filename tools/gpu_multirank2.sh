# cfg2 bench at 2 ranks on the box's one GPU (gloo): the N>1 path after the round-2 engine changes
export KVF_BENCH_ONE_DEVICE=1 KVF_BENCH_BACKEND=gloo
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29611 \
  bench.py --gpus 2 --steps 3 --warmup 3 --skip-decode --skip-configs --skip-cpu > gpurun_out/mr_cfg2.json 2> gpurun_out/mr_cfg2.err
echo "cfg2 2-rank rc=$?"; tail -c 2500 gpurun_out/mr_cfg2.json; tail -5 gpurun_out/mr_cfg2.err
