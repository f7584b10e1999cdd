D=gpurun_out/r02c5m; mkdir -p $D
for rep in 1 2; do for P in 2 4; do for mode in 2 0; do
  SPMAT_BSR_FUSE=$mode python -m torch.distributed.run --nnodes=1 --nproc-per-node $P --master-addr 127.0.0.1 --master-port 2969$P bench.py --gpus $P --config c5 --steps 20 --warmup 5 --no-cpu --no-e2e > $D/c5_p${P}_m${mode}_$rep.json 2> $D/c5_p${P}_m${mode}_$rep.err
  python -c "
import json; d=json.loads(open('$D/c5_p${P}_m${mode}_$rep.json').read().strip().splitlines()[-1]); print('P=$P mode=$mode rep=$rep', round(d['ms_per_step'],4), [round(t,4) for t in d['trials_ms_per_step']], d['gpu_launches'], d['clocks']['sm_mhz'], d['clocks']['reasons'])" || tail -4 $D/c5_p${P}_m${mode}_$rep.err
done; done; done
timeout 1200 python -m pytest tests/test_gpu_multirank.py -rA -q -p no:cacheprovider -k "offdiag_3x3" > $D/pytest_3x3.log 2>&1; tail -9 $D/pytest_3x3.log
