# 4-GPU: C5 fused 3x3 off-diagonal at P=2,4 (vs the standalone kernel), multirank 3x3 tests, NVLink probe
D=gpurun_out/r02g4c; mkdir -p $D
python bench.py --config c5 --no-cpu --no-e2e --steps 50 > $D/c5_p1.json 2> $D/c5_p1.err
for P in 2 4; do
  python -m torch.distributed.run --nnodes=1 --nproc-per-node $P --master-addr 127.0.0.1 --master-port 2969$P bench.py --gpus $P --config c5 --no-cpu --no-e2e --steps 50 > $D/c5_p$P.json 2> $D/c5_p$P.err
  SPMAT_BSR_FUSE=0 python -m torch.distributed.run --nnodes=1 --nproc-per-node $P --master-addr 127.0.0.1 --master-port 2968$P bench.py --gpus $P --config c5 --no-cpu --no-e2e --steps 50 > $D/c5_p${P}_nofuse.json 2> $D/c5_p${P}_nofuse.err
done
for f in $D/*.json; do python -c "
import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', round(d['ms_per_step'],4), [round(t,4) for t in d['trials_ms_per_step']], round(d['value'],1), round(d['roofline']['frac'],3), 'setv_ms', round(d['assembly']['set_values_coo_ms'],3), d['phases_ms']['isolated'], d.get('halo'))" 2>/dev/null || (echo "$f failed"; tail -5 ${f%.json}.err); done
timeout 900 python -m pytest tests/test_gpu_multirank.py -rA -q -p no:cacheprovider -k "offdiag_3x3" > $D/pytest_3x3.log 2>&1; tail -8 $D/pytest_3x3.log
timeout 300 python tools/nvlink_probe.py > $D/nvlink_probe.log 2>&1; cat $D/nvlink_probe.log | tail -7
