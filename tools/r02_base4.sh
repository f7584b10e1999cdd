# round-2 baseline on 4 GPUs: raw GPU test log + C5/C4 bench lines before any change
D=gpurun_out/r02base; mkdir -p $D
git_sha=$(cat .tip_sha 2>/dev/null); echo "tip $git_sha" > $D/pytest.log
nvidia-smi -L >> $D/pytest.log
timeout 1300 python -m pytest tests -m gpu -rA -q -p no:cacheprovider >> $D/pytest.log 2>&1; tail -3 $D/pytest.log
for P in 1 2 4; do
  if [ $P = 1 ]; then python bench.py --config c5 --no-cpu --no-e2e > $D/c5_p1.json 2> $D/c5_p1.err
  else python -m torch.distributed.run --nnodes=1 --nproc-per-node $P --master-addr 127.0.0.1 --master-port 2969$P bench.py --gpus $P --config c5 --no-cpu --no-e2e > $D/c5_p$P.json 2> $D/c5_p$P.err; fi
done
python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29694 bench.py --gpus 4 --config c4b --no-cpu --no-e2e > $D/c4b_p4.json 2> $D/c4b_p4.err
for f in $D/*.json; do python -c "
import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', round(d['ms_per_step'],4), round(d['value'],1), round(d['roofline']['frac'],3), d['phases_ms'])" 2>/dev/null || echo "$f failed"; done
