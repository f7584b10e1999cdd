D=gpurun_out/r02fold2; mkdir -p $D
MP_CASES=full-c4b,box timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29652 tests/mp_gpu_parity.py > $D/mp_c4b_p2.log 2>&1; grep -E "FAIL|MULTI" $D/mp_c4b_p2.log | tail -3
for f in 1 0; do
SPMAT_TAIL_FOLD=$f SPMAT_TRACE=1 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29631 tools/trace_mult.py --config c4b --graph > $D/trace_fold$f.log 2>&1; echo "== fold $f"; grep -v "^\[W\|Warning\|warn\|\*\*\*\|OMP\|NCCL" $D/trace_fold$f.log | tail -4
done
python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e > $D/c4_p1.json 2> $D/c4_p1.err; python -c "
import json; d=json.loads(open('$D/c4_p1.json').read().strip().splitlines()[-1]); print('c4 P=1', round(d['ms_per_step'],4), round(d['roofline']['frac'],3))"
for f in 1 0; do SPMAT_TAIL_FOLD=$f python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29661 bench.py --gpus 2 --config c4b --steps 50 --warmup 5 --no-cpu --no-e2e > $D/c4b_p2_f$f.json 2> $D/c4b_p2_f$f.err; python -c "
import json; d=json.loads(open('$D/c4b_p2_f$f.json').read().strip().splitlines()[-1]); print('c4b P=2 fold $f', round(d['ms_per_step'],4), [round(t,4) for t in d['trials_ms_per_step']], d['clocks']['reasons'])"; done
