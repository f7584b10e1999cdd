# 4-GPU: C5 with the 3x3 off-diagonal kernel at P=1,2,4, then the multirank suite
D=gpurun_out/r02g4; mkdir -p $D
for P in 2 4; do
  python -m torch.distributed.run --nnodes=1 --nproc-per-node $P --master-addr 127.0.0.1 --master-port 2969$P bench.py --gpus $P --config c5 --no-cpu --no-e2e --steps 50 > $D/c5_p$P.json 2> $D/c5_p$P.err
  SPMAT_BSR_OFFDIAG=0 python -m torch.distributed.run --nnodes=1 --nproc-per-node $P --master-addr 127.0.0.1 --master-port 2968$P bench.py --gpus $P --config c5 --no-cpu --no-e2e --steps 50 > $D/c5_p${P}_csroff.json 2> $D/c5_p${P}_csroff.err
done
for f in $D/*.json; do python -c "
import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', round(d['ms_per_step'],4), round(d['value'],1), round(d['roofline']['frac'],3), d['phases_ms'], d.get('halo'))" 2>/dev/null || (echo "$f failed"; tail -5 ${f%.json}.err); done
timeout 1500 python -m pytest tests/test_gpu_multirank.py -rA -q -p no:cacheprovider -x > $D/pytest_mr.log 2>&1; tail -15 $D/pytest_mr.log
