# latency checks of the NVLink halo / scalar board (2 GPUs)
set -x
mkdir -p gpurun_out; timeout 1200 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/lat_pytest.log 2>&1; tail -3 gpurun_out/lat_pytest.log
timeout 300 python tools/cg_bench.py --configs kuu,bump --breakdown --iters 200 2>&1 | grep us/iter; SPMAT_PDL=0 timeout 300 python tools/cg_bench.py --configs kuu --breakdown --iters 200 2>&1 | grep us/iter
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29681 tools/cg_bench.py --configs kuu,bump,c4 --breakdown --iters 200 2>&1 | grep "us/iter"
for c in kuu bump; do SPMAT_TRACE=1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29684 tools/trace_mult.py --config $c --graph 2>&1 | grep -A3 "^rank"; done
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29682 bench.py --gpus 2 --steps 200 --warmup 10 --no-e2e 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print('P2 c4', round(d['value'],1), round(d['ms_per_step'],4))"
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29683 bench.py --gpus 2 --steps 50 --warmup 5 --no-e2e --config c5 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print('P2 c5', round(d['value'],1), round(d['ms_per_step'],4))"
