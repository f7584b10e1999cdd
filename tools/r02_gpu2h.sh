D=gpurun_out/r02g2h; mkdir -p $D
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "host_pipeline or cuda_graphs or vec_dot" > $D/pytest.log 2>&1; tail -2 $D/pytest.log
MP_CASES=host,cg python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29641 tests/mp_gpu_parity.py > $D/mp.log 2>&1; grep -E "PASS|FAIL|MULTI" $D/mp.log | tail -5
python bench.py --steps 20 --warmup 5 --no-cpu > $D/c4_p1.json 2> $D/c4_p1.err
python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29692 bench.py --gpus 2 --steps 20 --warmup 5 > $D/c4_p2.json 2> $D/c4_p2.err
for f in $D/*.json; do python -c "
import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', round(d['ms_per_step'],4), d['e2e'])" 2>/dev/null || (echo "$f failed"; tail -5 ${f%.json}.err); done
