# device traces of the fused MatMult kernel (graph replay), P=1 and P=2
for c in ${CONFIGS:-c4 kuu}; do
  echo "== $c P=1"; SPMAT_TRACE=1 timeout 300 python tools/trace_mult.py --config $c --graph 2>&1 | grep -A3 "^rank"
  echo "== $c P=2"; SPMAT_TRACE=1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29684 tools/trace_mult.py --config $c --graph 2>&1 | grep -A3 "^rank"
done
