# A/B of two library builds in one call: _ab/base.so vs the in-tree build (KVF_LIB)
# usage: bash tools/gpu_ab_lib.sh "<breakdown args>" "<env>"
ARGS="$1"; ENVS="$2"
for v in base new base new; do
  if [ "$v" = base ]; then LIB=_ab/base.so; else LIB=paper_2601_03067_b200/_lib/libkvfuse_b200.so; fi
  env $ENVS KVF_LIB=$LIB timeout 900 python tools/step_breakdown.py $ARGS > gpurun_out/ab_$v.txt 2>&1
  echo "$v: $(head -1 gpurun_out/ab_$v.txt | sed 's/.*step/step/')  sim $(sed -n 2p gpurun_out/ab_$v.txt | awk '{print $1}')"
done
