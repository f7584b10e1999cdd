# Row-block budget sized for one consumer pass (auto) vs the fixed 2048 (SPMAT_RB_BUDGET=0).
D=gpurun_out/r02bud; mkdir -p $D
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "full_size or kernel or long_rows or every_row or small" > $D/pytest.log 2>&1; tail -1 $D/pytest.log
for rep in 1 2; do for cfg in c2 c3 bump q2 c4; do for b in auto 0; do
  if [ $b = auto ]; then E="X=1"; else E="SPMAT_RB_BUDGET=0"; fi
  env $E python bench.py --config $cfg --steps 50 --warmup 5 --no-cpu --no-e2e > $D/${cfg}_$b.json 2> $D/${cfg}_$b.err
  python -c "
import json; d=json.loads(open('$D/${cfg}_$b.json').read().strip().splitlines()[-1]); r=d['roofline']; print('$cfg $b', round(d['ms_per_step'],4), round(r['frac'],3), round(r['avg_launch_ms'],4), d['clocks']['reasons'])" || tail -3 $D/${cfg}_$b.err
done; done; done
