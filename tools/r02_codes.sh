# One-byte column codes in the bulk-copy SpMV: parity, then A/B against int32 columns.
D=gpurun_out/r02codes; mkdir -p $D
timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider > $D/pytest.log 2>&1; tail -1 $D/pytest.log
for rep in 1 2; do for cfg in c4 c3 c2 q2 bump c4b; do for cc in 1 0; do
  SPMAT_COL_CODES=$cc python bench.py --config $cfg --steps 50 --warmup 5 --no-cpu --no-e2e > $D/${cfg}_$cc.json 2> $D/${cfg}_$cc.err
  python -c "
import json; d=json.loads(open('$D/${cfg}_$cc.json').read().strip().splitlines()[-1]); r=d['roofline']; print('$cfg codes=$cc', round(d['ms_per_step'],4), round(r['frac'],3), d['clocks']['reasons'])" || tail -3 $D/${cfg}_$cc.err
done; done; done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_spmv_tma -s 3 -c 1 -o $D/c4_codes python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --eager > $D/ncu.log 2>&1; tail -1 $D/ncu.log
