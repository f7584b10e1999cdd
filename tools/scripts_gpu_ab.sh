# A/B comparison of libspmat builds in paper_2406_08646_b200/_ab (same box, interleaved):
#   VARIANTS="a b" CONFIGS="c4 c4b" PS="1 2" bash tools/scripts_gpu_ab.sh
for rep in 1 2; do
for v in ${VARIANTS:-base}; do
  L=paper_2406_08646_b200/_ab/$v.so
  for cfg in ${CONFIGS:-c4}; do
    for P in ${PS:-2}; do
      if [ "$P" = 1 ]; then
        b=$(env SPMAT_LIB=$L $ENVS python bench.py --config $cfg --no-e2e --no-cpu 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print(round(d['ms_per_step']*1e3,1))")
      else
        b=$(env SPMAT_LIB=$L $ENVS python -m torch.distributed.run --nnodes=1 --nproc-per-node $P --master-addr 127.0.0.1 --master-port 29682 bench.py --gpus $P --config $cfg --no-e2e --no-cpu 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print(round(d['ms_per_step']*1e3,1))")
      fi
      echo "$v $ENVS: $cfg P$P $b us"
    done
  done
done; done
