# 4-GPU: box split tail A/B, box parity in both tail modes, C4 weak scaling refresh
D=gpurun_out/r02g4e; mkdir -p $D
python bench.py --config c4 --no-cpu --no-e2e --steps 100 > $D/c4_p1.json 2> $D/c4_p1.err
python bench.py --config c4b --no-cpu --no-e2e --steps 100 > $D/c4b_p1.json 2> $D/c4b_p1.err
for P in 2 4; do
  python -m torch.distributed.run --nnodes=1 --nproc-per-node $P --master-addr 127.0.0.1 --master-port 2969$P bench.py --gpus $P --config c4b --no-cpu --no-e2e --steps 100 > $D/c4b_p$P.json 2> $D/c4b_p$P.err
  SPMAT_SPLIT_TAIL=0 python -m torch.distributed.run --nnodes=1 --nproc-per-node $P --master-addr 127.0.0.1 --master-port 2968$P bench.py --gpus $P --config c4b --no-cpu --no-e2e --steps 100 > $D/c4b_p${P}_old.json 2> $D/c4b_p${P}_old.err
  python -m torch.distributed.run --nnodes=1 --nproc-per-node $P --master-addr 127.0.0.1 --master-port 2967$P bench.py --gpus $P --config c4 --no-cpu --no-e2e --steps 100 > $D/c4_p$P.json 2> $D/c4_p$P.err
done
for f in $D/*.json; do python -c "
import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', d.get('launch'), round(d['ms_per_step'],4), [round(t,4) for t in d['trials_ms_per_step']], round(d['value'],1), round(d['roofline']['frac'],3), d['phases_ms']['isolated'], d['clocks']['sm_mhz'], d['clocks']['reasons'])" 2>/dev/null || (echo "$f failed"; tail -5 ${f%.json}.err); done
for P in 2 4; do
  MP_CASES=box,stencil,host python -m torch.distributed.run --nnodes=1 --nproc-per-node $P --master-addr 127.0.0.1 --master-port 2966$P tests/mp_gpu_parity.py > $D/mp_box_p$P.log 2>&1; grep -E "PASS|FAIL|MULTIRANK" $D/mp_box_p$P.log | tail -8
  SPMAT_SPLIT_TAIL=1 MP_CASES=stencil,elasticity python -m torch.distributed.run --nnodes=1 --nproc-per-node $P --master-addr 127.0.0.1 --master-port 2965$P tests/mp_gpu_parity.py > $D/mp_split_p$P.log 2>&1; grep -E "FAIL|MULTIRANK" $D/mp_split_p$P.log | tail -3
done
