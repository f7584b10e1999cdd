# Element-COO numeric: the pipelined kernel as default, single- and multi-rank parity, C3 A/B.
D=gpurun_out/r02np; mkdir -p $D
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "numeric or block_csr or full_size" > $D/pytest.log 2>&1; tail -1 $D/pytest.log
MP_CASES=q1,random,elasticity python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29641 tests/mp_gpu_parity.py > $D/mp.log 2>&1; grep -E "FAIL|MULTI" $D/mp.log | tail -3
for k in seg pipe2 seg pipe2; do SPMAT_NUMERIC_KERNEL=$k python bench.py --config c3 --no-cpu --no-e2e --steps 5 > $D/c3_$k.json 2> $D/c3_$k.err
python -c "
import json; d=json.loads(open('$D/c3_$k.json').read().strip().splitlines()[-1]); print('$k', 'setv_ms', round(d['assembly']['set_values_coo_ms'],4))"; done
for k in seg pipe2; do SPMAT_NUMERIC_KERNEL=$k python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29642 bench.py --gpus 2 --config c3 --no-cpu --no-e2e --steps 5 > $D/c3p2_$k.json 2> $D/c3p2_$k.err
python -c "
import json; d=json.loads(open('$D/c3p2_$k.json').read().strip().splitlines()[-1]); print('P=2 $k', 'setv_ms', round(d['assembly']['set_values_coo_ms'],4))"; done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_numeric_seg_pipe -c 1 -o $D/c3_pipe2 python bench.py --config c3 --no-cpu --no-e2e --steps 3 --warmup 3 > $D/ncu.log 2>&1; tail -1 $D/ncu.log
