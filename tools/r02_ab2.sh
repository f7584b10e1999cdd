D=gpurun_out/r02ab2; mkdir -p $D
for c in 1 2 4 8; do SPMAT_PIPE_CHUNKS_ASYNC=$c python bench.py --steps 20 --warmup 5 --no-cpu > $D/c4_async$c.json 2> $D/c4_async$c.err
python -c "
import json; d=json.loads(open('$D/c4_async$c.json').read().strip().splitlines()[-1]); e=d['e2e']; print('async chunks $c', round(e['ms_per_step'],3), round(e['value'],1), 'sync', round(e['sync_call_ms_per_step'],3), e['y_equals_device_result'])"; done
for f in 0 1 0 1; do SPMAT_BSR_FMA=$f python bench.py --config c5 --steps 20 --warmup 5 --no-cpu --no-e2e > $D/c5_fma$f.json 2> $D/c5_fma$f.err
python -c "
import json; d=json.loads(open('$D/c5_fma$f.json').read().strip().splitlines()[-1]); print('c5 fma=$f', round(d['ms_per_step'],4), [round(t,4) for t in d['trials_ms_per_step']], round(d['roofline']['frac'],3), d['clocks']['sm_mhz'], d['clocks']['reasons'])"; done
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "block_csr or full_size or host_pipeline" > $D/pytest.log 2>&1; tail -1 $D/pytest.log
SPMAT_BSR_FMA=1 timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "block_csr or full_size" > $D/pytest_fma.log 2>&1; tail -1 $D/pytest_fma.log
