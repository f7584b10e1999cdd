D=gpurun_out/r02g2j; mkdir -p $D
for mode in 1 0 2 1; do for cfg in c4 c4b; do
  SPMAT_COOP=$mode python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 2969$mode bench.py --gpus 2 --config $cfg --no-cpu --no-e2e --steps 20 > $D/${cfg}_coop$mode.json 2> $D/${cfg}_coop$mode.err
  python -c "
import json,sys; d=json.loads(open('$D/${cfg}_coop$mode.json').read().strip().splitlines()[-1]); print('$cfg coop=$mode', d.get('launch'), round(d['ms_per_step'],4), [round(t,4) for t in d['trials_ms_per_step']], d['clocks']['sm_mhz'], d['clocks']['reasons'])" || tail -5 $D/${cfg}_coop$mode.err
done; done
python bench.py --config c4 --no-cpu --no-e2e --steps 20 > $D/c4_p1.json 2>&1; python -c "
import json; d=json.loads(open('$D/c4_p1.json').read().strip().splitlines()[-1]); print('c4 P=1', round(d['ms_per_step'],4), [round(t,4) for t in d['trials_ms_per_step']])"
