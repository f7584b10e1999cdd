# Split tail with the consumer fold: parity (small cases forced through the tma kernel, the
# full-size C4b case at P=2 and 4), then C4b weak scaling A/B (fold on/off) and C4 P=1 check.
D=gpurun_out/r02fold; mkdir -p $D
timeout 1200 python -m pytest tests/test_gpu_multirank.py -m gpu -q -x -p no:cacheprovider -k "tma_tails" > $D/pytest_tails.log 2>&1; tail -1 $D/pytest_tails.log
for P in 2 4; do MP_CASES=full-c4b,box timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $P --master-addr 127.0.0.1 --master-port 2965$P tests/mp_gpu_parity.py > $D/mp_c4b_p$P.log 2>&1; grep -E "FAIL|MULTI" $D/mp_c4b_p$P.log | tail -3; done
run() {  # name P env...
  n=$1; P=$2; shift 2
  if [ $P = 1 ]; then env "$@" python bench.py --config c4b --steps 50 --warmup 5 --no-cpu --no-e2e > $D/$n.json 2> $D/$n.err
  else env "$@" python -m torch.distributed.run --nnodes=1 --nproc-per-node $P --master-addr 127.0.0.1 --master-port 29661 bench.py --gpus $P --config c4b --steps 50 --warmup 5 --no-cpu --no-e2e > $D/$n.json 2> $D/$n.err; fi
  python -c "
import json; d=json.loads(open('$D/$n.json').read().strip().splitlines()[-1]); print('$n', round(d['ms_per_step'],4), [round(t,4) for t in d['trials_ms_per_step']], d['clocks']['sm_mhz'], d['clocks']['reasons'], d['phases_ms'].get('overlap_efficiency'))" || tail -3 $D/$n.err
}
run c4b_p1 1 X=1
for rep in 1 2; do
run c4b_p4_fold_$rep 4 SPMAT_TAIL_FOLD=1
run c4b_p4_nofold_$rep 4 SPMAT_TAIL_FOLD=0
run c4b_p2_fold_$rep 2 SPMAT_TAIL_FOLD=1
run c4b_p2_nofold_$rep 2 SPMAT_TAIL_FOLD=0
done
run c4b_p1_b 1 X=1
python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e > $D/c4_p1.json 2> $D/c4_p1.err; python -c "
import json; d=json.loads(open('$D/c4_p1.json').read().strip().splitlines()[-1]); print('c4 P=1', round(d['ms_per_step'],4), round(d['roofline']['frac'],3))"
