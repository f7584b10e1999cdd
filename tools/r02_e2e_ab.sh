D=gpurun_out/r02e2e; mkdir -p $D
python tools/pcie_bench.py > $D/pcie.log 2>&1; tail -4 $D/pcie.log
for c in 8 16 32 64; do SPMAT_PIPE_CHUNKS=$c python bench.py --steps 20 --warmup 5 --no-cpu > $D/c4_chunks$c.json 2> $D/c4_chunks$c.err
python -c "
import json; d=json.loads(open('$D/c4_chunks$c.json').read().strip().splitlines()[-1]); e=d['e2e']; print('chunks $c', round(e['ms_per_step'],3), round(e['value'],1), round(e['sync_call_ms_per_step'],3), e['y_equals_device_result'])"; done
