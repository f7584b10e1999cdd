# A/B comparison of libspmat builds in paper_2406_08646_b200/_ab (same box, interleaved)
for rep in 1 2; do
for v in ${VARIANTS:-cons nocons smem}; do
  L=paper_2406_08646_b200/_ab/$v.so
  a=$(SPMAT_LIB=$L python bench.py --no-e2e --no-cpu 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print(round(d['ms_per_step']*1e3,1))")
  b=$(SPMAT_LIB=$L python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29682 bench.py --gpus 2 --no-e2e --no-cpu 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print(round(d['ms_per_step']*1e3,1))")
  c=$(SPMAT_LIB=$L python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29683 tools/cg_bench.py --configs kuu,bump --breakdown --iters 200 2>&1 | grep us/iter | awk '{print $1, $5, "mult", $8}' | tr '\n' ' ')
  echo "$v: c4 P1 $a us, P2 $b us; CG P2: $c"
done; done
