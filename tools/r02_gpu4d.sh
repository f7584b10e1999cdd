# 4-GPU: box decomposition (progressive tail) A/B at P=2,4; multirank parity; SF pingpong breakdown; C1 graph
D=gpurun_out/r02g4d; mkdir -p $D
python bench.py --config c1 --no-cpu --no-e2e --steps 200 > $D/c1_p1.json 2> $D/c1_p1.err
python bench.py --config c4b --no-cpu --no-e2e --steps 50 > $D/c4b_p1.json 2> $D/c4b_p1.err
for P in 2 4; do
  python -m torch.distributed.run --nnodes=1 --nproc-per-node $P --master-addr 127.0.0.1 --master-port 2969$P bench.py --gpus $P --config c4b --no-cpu --no-e2e --steps 50 > $D/c4b_p$P.json 2> $D/c4b_p$P.err
  SPMAT_PROGRESSIVE_TAIL=0 python -m torch.distributed.run --nnodes=1 --nproc-per-node $P --master-addr 127.0.0.1 --master-port 2968$P bench.py --gpus $P --config c4b --no-cpu --no-e2e --steps 50 > $D/c4b_p${P}_old.json 2> $D/c4b_p${P}_old.err
done
python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29664 bench.py --gpus 4 --config c4 --no-cpu --no-e2e --steps 50 > $D/c4_p4.json 2> $D/c4_p4.err
for f in $D/*.json; do python -c "
import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', d.get('launch'), round(d['ms_per_step'],4), [round(t,4) for t in d['trials_ms_per_step']], round(d['value'],1), round(d['roofline']['frac'],3), d['phases_ms']['isolated'], d['clocks']['sm_mhz'], d['clocks']['reasons'])" 2>/dev/null || (echo "$f failed"; tail -5 ${f%.json}.err); done
timeout 1200 python -m pytest tests/test_gpu_multirank.py -rA -q -p no:cacheprovider -k "parity" > $D/pytest_mr.log 2>&1; tail -6 $D/pytest_mr.log
python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29655 tools/sf_bench.py --graph --breakdown > $D/sf_pingpong_graph.log 2>&1; tail -14 $D/sf_pingpong_graph.log
SPMAT_SF=nccl python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29656 tools/sf_bench.py --breakdown > $D/sf_pingpong_nccl.log 2>&1; tail -3 $D/sf_pingpong_nccl.log
