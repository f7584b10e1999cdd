D=gpurun_out/r02tr; mkdir -p $D
for cfg in c4 c4b; do
SPMAT_TRACE=1 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29631 tools/trace_mult.py --config $cfg --graph > $D/trace_$cfg.log 2>&1; echo "== $cfg"; grep -v "^\[W\|Warning\|warn" $D/trace_$cfg.log | tail -8
done
