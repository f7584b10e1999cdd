# A/B of the element-COO numeric kernels on C3 (k_numeric_seg vs the lean variants), then one
# ncu --set full capture of the lean kernel.
D=gpurun_out/r02nl; mkdir -p $D
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "numeric" > $D/pytest.log 2>&1; tail -1 $D/pytest.log
for k in pipe4 pipe2 pipe2s pipe1 pipe3 pipe4 pipe2 pipe2s pipe1 pipe3; do SPMAT_NUMERIC_KERNEL=$k python bench.py --config c3 --no-cpu --no-e2e --steps 5 > $D/c3_$k.json 2> $D/c3_$k.err
python -c "
import json; d=json.loads(open('$D/c3_$k.json').read().strip().splitlines()[-1]); print('$k', 'setv_ms', round(d['assembly']['set_values_coo_ms'],4))"; done
SPMAT_NUMERIC_KERNEL=pipe2s timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_numeric_seg -c 1 -o $D/c3_lean python bench.py --config c3 --no-cpu --no-e2e --steps 3 --warmup 3 > $D/ncu.log 2>&1; tail -2 $D/ncu.log
