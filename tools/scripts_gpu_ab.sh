# A/B comparison of libspmat builds in paper_2406_08646_b200/_ab (same box, interleaved):
#   VARIANTS="a b" CONFIG=c4b ENVS="X=1" bash tools/scripts_gpu_ab.sh
for rep in 1 2; do
for v in ${VARIANTS:-base}; do
  L=paper_2406_08646_b200/_ab/$v.so
  for cfg in ${CONFIGS:-c4}; do
    b=$(env SPMAT_LIB=$L $ENVS python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29682 bench.py --gpus 2 --config $cfg --no-e2e --no-cpu 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print(round(d['ms_per_step']*1e3,1))")
    echo "$v $ENVS: $cfg P2 $b us"
  done
done; done
