# 2 GPUs: GPU parity (1 GPU), numeric + MatMult lines C2-C5, CG table, SF pingpong with the new bulk protocol
D=gpurun_out/r02g2f; mkdir -p $D
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider > $D/pytest.log 2>&1; tail -2 $D/pytest.log
for cfg in c2 c3 c4 c5; do python bench.py --config $cfg --no-cpu --no-e2e --steps 20 > $D/${cfg}_p1.json 2> $D/${cfg}_p1.err; done
for f in $D/*.json; do python -c "
import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', round(d['ms_per_step'],4), round(d['roofline']['frac'],3), 'setv_ms', round(d['assembly']['set_values_coo_ms'],3), round(d['assembly']['set_values_GBps'],1), d['clocks']['sm_mhz'], d['clocks']['reasons'])" 2>/dev/null || (echo "$f failed"; tail -5 ${f%.json}.err); done
python tools/cg_bench.py --configs kuu,bump,bump7 --breakdown --iters 100 > $D/cg_p1.log 2>&1; grep us/iter $D/cg_p1.log
python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29655 tools/sf_bench.py --graph --breakdown > $D/sf_pingpong_graph.log 2>&1; tail -13 $D/sf_pingpong_graph.log
timeout 600 python -m pytest tests/test_gpu_multirank.py -q -p no:cacheprovider -k "bulk or board" > $D/pytest_mr.log 2>&1; tail -2 $D/pytest_mr.log
