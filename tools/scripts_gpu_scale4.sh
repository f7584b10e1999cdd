# 4-GPU refresh: GPU tests, C4/C4b/C5 bench lines at P=1,2,4, host-pipeline A/B, CG at P=1,2,4
D=gpurun_out/scale4; mkdir -p $D
timeout 1300 python -m pytest tests -m gpu -q -x -p no:cacheprovider > $D/pytest.log 2>&1; tail -2 $D/pytest.log
for cfg in c4 c4b c5; do
  python bench.py --config $cfg --no-cpu > $D/${cfg}_p1.json 2> $D/${cfg}_p1.err
  for P in 2 4; do
    python -m torch.distributed.run --nnodes=1 --nproc-per-node $P --master-addr 127.0.0.1 --master-port 2969$P bench.py --gpus $P --config $cfg --no-cpu > $D/${cfg}_p$P.json 2> $D/${cfg}_p$P.err
  done
done
for P in 2 4; do
  SPMAT_HOST_PIPELINE=0 python -m torch.distributed.run --nnodes=1 --nproc-per-node $P --master-addr 127.0.0.1 --master-port 2968$P bench.py --gpus $P --no-cpu > $D/c4_p${P}_nopipe.json 2>/dev/null
done
python tools/cg_bench.py --configs kuu,bump,c4 --breakdown --iters 200 2>&1 | grep us/iter
for P in 2 4; do python -m torch.distributed.run --nnodes=1 --nproc-per-node $P --master-addr 127.0.0.1 --master-port 2967$P tools/cg_bench.py --configs kuu,bump,c4 --breakdown --iters 200 2>&1 | grep us/iter; done
for f in $D/*.json; do python -c "
import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', round(d['ms_per_step'],4), round(d['value'],1), round(d['roofline']['frac'],3), (d.get('e2e') or {}).get('value'))" 2>/dev/null || echo "$f failed"; done
