D=gpurun_out/r02nw; mkdir -p $D
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "numeric" > $D/pytest.log 2>&1; tail -1 $D/pytest.log
for k in seg warp seg warp; do SPMAT_NUMERIC_KERNEL=$k python bench.py --config c3 --no-cpu --no-e2e --steps 20 > $D/c3_$k.json 2> $D/c3_$k.err
python -c "
import json; d=json.loads(open('$D/c3_$k.json').read().strip().splitlines()[-1]); print('$k', 'setv_ms', round(d['assembly']['set_values_coo_ms'],4))"; done
SPMAT_NUMERIC_KERNEL=warp MP_CASES=q1,random python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29641 tests/mp_gpu_parity.py > $D/mp.log 2>&1; grep -E "FAIL|MULTI" $D/mp.log | tail -3
