# k_spmv_bsr3: cap on lanes per block row (SPMAT_BSR_WMAX), C5 at P=1 (power-capped) and P=4
D=gpurun_out/r02bsrw; mkdir -p $D
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "block_csr or c5" > $D/pytest.log 2>&1; tail -1 $D/pytest.log
for rep in 1 2; do for w in 32 8 4; do
  SPMAT_BSR_WMAX=$w python bench.py --config c5 --steps 20 --warmup 5 --no-cpu --no-e2e > $D/c5_w$w.json 2> $D/c5_w$w.err
  python -c "
import json; d=json.loads(open('$D/c5_w$w.json').read().strip().splitlines()[-1]); print('c5 P=1 wmax=$w', round(d['ms_per_step'],4), [round(t,4) for t in d['trials_ms_per_step']], d['clocks']['sm_mhz'], d['clocks']['reasons'])" || tail -3 $D/c5_w$w.err
done; done
for rep in 1 2; do for w in 32 8; do
  SPMAT_BSR_WMAX=$w python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29691 bench.py --gpus 4 --config c5 --steps 20 --warmup 5 --no-cpu --no-e2e > $D/c5p4_w$w.json 2> $D/c5p4_w$w.err
  python -c "
import json; d=json.loads(open('$D/c5p4_w$w.json').read().strip().splitlines()[-1]); print('c5 P=4 wmax=$w', round(d['ms_per_step'],4), [round(t,4) for t in d['trials_ms_per_step']], d['clocks']['sm_mhz'], d['clocks']['reasons'])" || tail -3 $D/c5p4_w$w.err
done; done
for w in 32 8; do SPMAT_BSR_WMAX=$w timeout 600 ncu --set full --clock-control none -k regex:k_spmv_bsr3 -s 2 -c 1 -o $D/c5_w$w python bench.py --config c5 --steps 3 --warmup 3 --no-cpu --no-e2e > $D/ncu_w$w.log 2>&1; tail -1 $D/ncu_w$w.log; done
