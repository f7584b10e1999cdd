D=gpurun_out/r02p3; mkdir -p $D
python -m torch.distributed.run --nnodes=1 --nproc-per-node 3 --master-addr 127.0.0.1 --master-port 29643 tests/mp_gpu_parity.py > $D/mp_p3.log 2>&1; grep -E "FAIL|MULTI" $D/mp_p3.log | tail -5
SPMAT_HALO=nccl python -m torch.distributed.run --nnodes=1 --nproc-per-node 3 --master-addr 127.0.0.1 --master-port 29644 tests/mp_gpu_parity.py > $D/mp_p3_nccl.log 2>&1; grep -E "FAIL|MULTI" $D/mp_p3_nccl.log | tail -5
for cfg in c4 c5; do python -m torch.distributed.run --nnodes=1 --nproc-per-node 3 --master-addr 127.0.0.1 --master-port 29645 bench.py --gpus 3 --config $cfg --steps 20 --warmup 5 --no-cpu --no-e2e > $D/${cfg}_p3.json 2> $D/${cfg}_p3.err
python -c "
import json; d=json.loads(open('$D/${cfg}_p3.json').read().strip().splitlines()[-1]); print('$cfg P=3', round(d['ms_per_step'],4), round(d['value'],1), d['clocks']['sm_mhz'], d['clocks']['reasons'])" || tail -5 $D/${cfg}_p3.err; done
