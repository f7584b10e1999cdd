D=gpurun_out/r02pipe; mkdir -p $D
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "host_pipeline" > $D/pytest.log 2>&1; tail -1 $D/pytest.log
MP_CASES=host python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29641 tests/mp_gpu_parity.py > $D/mp.log 2>&1; grep -E "PASS|FAIL|MULTI" $D/mp.log | tail -4
for k in 1 2; do python bench.py --steps 20 --warmup 5 --no-cpu > $D/c4_p1_$k.json 2> $D/c4_p1_$k.err
python -c "
import json; d=json.loads(open('$D/c4_p1_$k.json').read().strip().splitlines()[-1]); e=d['e2e']; print('P=1', round(e['ms_per_step'],3), round(e['value'],1), 'async', round(e['async_call_ms_per_step'],3), 'sync', round(e['sync_call_ms_per_step'],3), e['y_equals_device_result'])"; done
python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29692 bench.py --gpus 2 --steps 20 --warmup 5 --no-cpu > $D/c4_p2.json 2> $D/c4_p2.err
python -c "
import json; d=json.loads(open('$D/c4_p2.json').read().strip().splitlines()[-1]); e=d['e2e']; print('P=2', round(e['ms_per_step'],3), round(e['value'],1), 'async', round(e['async_call_ms_per_step'],3), 'sync', round(e['sync_call_ms_per_step'],3), e['y_equals_device_result'])"
