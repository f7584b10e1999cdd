# Split tail with the add pass prefetched before the sweep-end wait: parity + C4b A/B.
D=gpurun_out/r02tail3; mkdir -p $D
timeout 1200 python -m pytest tests/test_gpu_multirank.py -m gpu -q -x -p no:cacheprovider -k "tma_tails" > $D/pytest_tails.log 2>&1; tail -1 $D/pytest_tails.log
for P in 2 4; do MP_CASES=full-c4b,box timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $P --master-addr 127.0.0.1 --master-port 2965$P tests/mp_gpu_parity.py > $D/mp_c4b_p$P.log 2>&1; grep -E "FAIL|MULTI" $D/mp_c4b_p$P.log | tail -3; done
SPMAT_TRACE=1 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29631 tools/trace_mult.py --config c4b --graph > $D/trace.log 2>&1; grep -v "^\[W\|Warning\|warn\|\*\*\*\|OMP\|NCCL" $D/trace.log | tail -4
run() {  # name P
  n=$1; P=$2
  if [ $P = 1 ]; then python bench.py --config c4b --steps 50 --warmup 5 --no-cpu --no-e2e > $D/$n.json 2> $D/$n.err
  else python -m torch.distributed.run --nnodes=1 --nproc-per-node $P --master-addr 127.0.0.1 --master-port 29661 bench.py --gpus $P --config c4b --steps 50 --warmup 5 --no-cpu --no-e2e > $D/$n.json 2> $D/$n.err; fi
  python -c "
import json; d=json.loads(open('$D/$n.json').read().strip().splitlines()[-1]); print('$n', round(d['ms_per_step'],4), [round(t,4) for t in d['trials_ms_per_step']], d['clocks']['sm_mhz'], d['clocks']['reasons'], d['phases_ms'].get('overlap_efficiency'), d['phases_ms'].get('isolated'))" || tail -3 $D/$n.err
}
run c4b_p1 1; run c4b_p2 2; run c4b_p4 4; run c4b_p1b 1; run c4b_p4b 4
