# 4-GPU refresh: GPU tests, C4/C4b/C5 bench lines at P=1,2,4, CG at P=4
mkdir -p gpurun_out/scale
timeout 1300 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/scale/pytest.log 2>&1; tail -2 gpurun_out/scale/pytest.log
for cfg in c4 c4b c5; do
  python bench.py --config $cfg --no-cpu > gpurun_out/scale/${cfg}_p1.json 2> gpurun_out/scale/${cfg}_p1.err
  for P in 2 4; do
    python -m torch.distributed.run --nnodes=1 --nproc-per-node $P --master-addr 127.0.0.1 --master-port 2969$P bench.py --gpus $P --config $cfg --no-cpu > gpurun_out/scale/${cfg}_p$P.json 2> gpurun_out/scale/${cfg}_p$P.err
  done
done
python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29699 tools/cg_bench.py --configs kuu,bump,c4 --breakdown --iters 200 2>&1 | grep us/iter
for f in gpurun_out/scale/*.json; do python -c "
import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', round(d['ms_per_step'],4), round(d['value'],1), round(d['roofline']['frac'],3), (d.get('e2e') or {}).get('value'))" 2>/dev/null || echo "$f failed"; done
