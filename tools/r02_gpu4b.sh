# 4-GPU box: parity of the new kernels (1 GPU), P=1 bench lines (C1/C3/C5), CG table, C5/C4/C4b at P=2,4
D=gpurun_out/r02g4b; mkdir -p $D
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider > $D/pytest.log 2>&1; tail -3 $D/pytest.log
for cfg in c1 c3 c5; do python bench.py --config $cfg --no-cpu --no-e2e --steps 50 > $D/${cfg}_p1.json 2> $D/${cfg}_p1.err; done
python tools/cg_bench.py --configs kuu,bump,bump7 --breakdown --iters 100 > $D/cg_p1.log 2>&1; grep us/iter $D/cg_p1.log
for P in 2 4; do
  python -m torch.distributed.run --nnodes=1 --nproc-per-node $P --master-addr 127.0.0.1 --master-port 2969$P bench.py --gpus $P --config c5 --no-cpu --no-e2e --steps 50 > $D/c5_p$P.json 2> $D/c5_p$P.err
  python -m torch.distributed.run --nnodes=1 --nproc-per-node $P --master-addr 127.0.0.1 --master-port 2967$P tools/cg_bench.py --configs kuu,bump --breakdown --iters 100 > $D/cg_p$P.log 2>&1; grep us/iter $D/cg_p$P.log
done
for cfg in c4 c4b; do python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29664 bench.py --gpus 4 --config $cfg --no-cpu --no-e2e --steps 50 > $D/${cfg}_p4.json 2> $D/${cfg}_p4.err; done
for f in $D/*.json; do python -c "
import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', round(d['ms_per_step'],4), round(d['value'],1), round(d['roofline']['frac'],3), d['roofline']['kernel'][:14], 'setv_ms', round(d['assembly']['set_values_coo_ms'],3), d['phases_ms'], (d.get('halo') or {}).get('halo_nvlink_frac'))" 2>/dev/null || (echo "$f failed"; tail -5 ${f%.json}.err); done
