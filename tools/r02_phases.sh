# Isolated phases launched like the headline trials (CUDA graphs): overlap_efficiency check.
D=gpurun_out/r02ph; mkdir -p $D
for spec in "c4:2" "c4b:4" "c5:4" "c5:2"; do IFS=: read cfg P <<< "$spec"
  python -m torch.distributed.run --nnodes=1 --nproc-per-node $P --master-addr 127.0.0.1 --master-port 29691 bench.py --gpus $P --config $cfg --steps 20 --warmup 5 --no-cpu --no-e2e > $D/${cfg}_p$P.json 2> $D/${cfg}_p$P.err
  python -c "
import json; d=json.loads(open('$D/${cfg}_p$P.json').read().strip().splitlines()[-1]); ph=d['phases_ms']; print('$cfg P=$P', round(d['ms_per_step'],4), ph['isolated_launch'], {k: round(v,4) for k,v in ph['isolated'].items()}, round(ph['overlap_efficiency'],3))" || tail -5 $D/${cfg}_p$P.err
done
