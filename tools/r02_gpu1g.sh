D=gpurun_out/r02g1g; mkdir -p $D
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "block_csr or numeric or full_size" > $D/pytest.log 2>&1; tail -2 $D/pytest.log
for cfg in c5 c4; do python bench.py --config $cfg --no-cpu --no-e2e --steps 20 > $D/${cfg}_p1.json 2> $D/${cfg}_p1.err; done
for f in $D/*.json; do python -c "
import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', round(d['ms_per_step'],4), round(d['roofline']['frac'],3), 'setv_ms', round(d['assembly']['set_values_coo_ms'],3), round(d['assembly']['set_values_GBps'],1), d['clocks']['sm_mhz'], d['clocks']['reasons'])" 2>/dev/null || (echo "$f failed"; tail -5 ${f%.json}.err); done
