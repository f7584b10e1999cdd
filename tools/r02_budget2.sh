D=gpurun_out/r02bud2; mkdir -p $D
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "full_size or kernel or long_rows or every_row or small" > $D/pytest.log 2>&1; tail -1 $D/pytest.log
for cfg in c3 c2 q2 bump; do python bench.py --config $cfg --steps 50 --warmup 5 --no-cpu --no-e2e > $D/${cfg}.json 2> $D/${cfg}.err
  python -c "
import json; d=json.loads(open('$D/${cfg}.json').read().strip().splitlines()[-1]); r=d['roofline']; print('$cfg', round(d['ms_per_step'],4), round(r['frac'],3), round(r['avg_launch_ms'],4), d['clocks']['reasons'])" || tail -3 $D/${cfg}.err; done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_spmv_tma -s 3 -c 1 -o $D/c3_tma python bench.py --config c3 --steps 3 --warmup 3 --no-cpu --no-e2e --eager > $D/ncu.log 2>&1; tail -1 $D/ncu.log
