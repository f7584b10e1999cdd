D=gpurun_out/r02one; mkdir -p $D
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "numeric or block_csr or full_size" > $D/pytest.log 2>&1; tail -1 $D/pytest.log
MP_CASES=stencil,random,elasticity,full-c4 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29641 tests/mp_gpu_parity.py > $D/mp.log 2>&1; grep -E "FAIL|MULTI" $D/mp.log | tail -3
for rep in 1 2; do for k in one ilp; do for cfg in c4 c5; do SPMAT_NUMERIC_KERNEL=$k python bench.py --config $cfg --no-cpu --no-e2e --steps 5 > $D/${cfg}_$k.json 2> $D/${cfg}_$k.err
python -c "
import json; d=json.loads(open('$D/${cfg}_$k.json').read().strip().splitlines()[-1]); print('$cfg $k', 'setv_ms', round(d['assembly']['set_values_coo_ms'],4))"; done; done; done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_numeric_one -c 1 -o $D/c4_one python bench.py --no-cpu --no-e2e --steps 3 --warmup 3 > $D/ncu.log 2>&1; tail -1 $D/ncu.log
