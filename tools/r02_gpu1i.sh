D=gpurun_out/r02g1i; mkdir -p $D
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "numeric" > $D/pytest.log 2>&1; tail -2 $D/pytest.log
python bench.py --config c3 --no-cpu --no-e2e --steps 20 > $D/c3_seg4.json 2> $D/c3_seg4.err
SPMAT_NUMERIC_SEG=8 python bench.py --config c3 --no-cpu --no-e2e --steps 20 > $D/c3_seg8.json 2> $D/c3_seg8.err
SPMAT_NUMERIC_KERNEL=plain python bench.py --config c3 --no-cpu --no-e2e --steps 20 > $D/c3_plain.json 2> $D/c3_plain.err
python bench.py --config c3 --no-cpu --no-e2e --steps 20 > $D/c3_seg4b.json 2> $D/c3_seg4b.err
for f in $D/*.json; do python -c "
import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', 'setv_ms', round(d['assembly']['set_values_coo_ms'],4), round(d['assembly']['set_values_GBps'],1), d['clocks']['sm_mhz'])" 2>/dev/null || (echo "$f failed"; tail -5 ${f%.json}.err); done
