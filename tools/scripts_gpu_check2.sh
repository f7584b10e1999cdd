# 2-GPU check: GPU tests, traces, P=1/P=2 bench lines (c4, c5), CG
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/c2_pytest.log 2>&1; tail -2 gpurun_out/c2_pytest.log
for cfg in c4 c5; do
python bench.py --config $cfg --no-e2e --no-cpu 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print('P1 $cfg', d['ms_per_step'], d['phases_ms']['isolated'])"
python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29682 bench.py --gpus 2 --config $cfg --no-e2e --no-cpu 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print('P2 $cfg', d['ms_per_step'], d['phases_ms'])"
done
python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29683 tools/cg_bench.py --configs kuu,bump --breakdown --iters 200 2>&1 | grep us/iter
