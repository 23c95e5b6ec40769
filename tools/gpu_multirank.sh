# multi-rank bench paths on the one GPU of a gpurun box (every rank on cuda:0, gloo):
# cfg5 layer-sharded (2 ranks x 1 full-shape layer) and cfg2 layer-sharded (2 ranks); then the
# single-rank cfg5 command for comparison
timeout 900 python bench.py --config cfg5 --layers-per-rank 2 --steps 1 --warmup 1 > gpurun_out/cfg5_1r.json 2> gpurun_out/cfg5_1r.err
echo "cfg5 1-rank rc=$?"; tail -c 1200 gpurun_out/cfg5_1r.json
export KVF_BENCH_ONE_DEVICE=1 KVF_BENCH_BACKEND=gloo
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29611 \
  bench.py --gpus 2 --config cfg5 --layers-per-rank 1 --steps 1 --warmup 1 > gpurun_out/mr_cfg5.json 2> gpurun_out/mr_cfg5.err
echo "cfg5 2-rank rc=$?"; tail -c 1500 gpurun_out/mr_cfg5.json
