D=gpurun_out/r02fma; mkdir -p $D
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "block_csr or full_size" > $D/pytest.log 2>&1; tail -1 $D/pytest.log
for f in 1 0 1 0; do SPMAT_BSR_FMA=$f python bench.py --config c5 --steps 20 --warmup 5 --no-cpu --no-e2e > $D/c5_p1_fma$f.json 2> $D/c5_p1_fma$f.err
python -c "
import json; d=json.loads(open('$D/c5_p1_fma$f.json').read().strip().splitlines()[-1]); print('P=1 fma=$f', round(d['ms_per_step'],4), [round(t,4) for t in d['trials_ms_per_step']], d['clocks']['sm_mhz'], d['clocks']['reasons'])"; done
for f in 1 0 1 0; do SPMAT_BSR_FMA=$f python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29694 bench.py --gpus 4 --config c5 --steps 20 --warmup 5 --no-cpu --no-e2e > $D/c5_p4_fma$f.json 2> $D/c5_p4_fma$f.err
python -c "
import json; d=json.loads(open('$D/c5_p4_fma$f.json').read().strip().splitlines()[-1]); print('P=4 fma=$f', round(d['ms_per_step'],4), [round(t,4) for t in d['trials_ms_per_step']], d['clocks']['sm_mhz'], d['clocks']['reasons'])"; done
timeout 900 python -m pytest tests/test_gpu_multirank.py -q -p no:cacheprovider -k "offdiag_3x3" > $D/pytest_mr.log 2>&1; tail -1 $D/pytest_mr.log
