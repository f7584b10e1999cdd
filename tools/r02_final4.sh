# Round-2 final evidence on 4 GPUs (run at the tip; results copied into profiles/ by hand)
D=gpurun_out/${R02_OUT:-r02final}; mkdir -p $D
{ echo "tip: $(cat .tip_sha 2>/dev/null)"; date -u; nvidia-smi -L; } > $D/pytest_gpu_4gpu.log
timeout 2400 python -m pytest tests -m gpu -rA -p no:cacheprovider >> $D/pytest_gpu_4gpu.log 2>&1; echo "pytest rc=$?"; tail -3 $D/pytest_gpu_4gpu.log
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $D/smoke.log 2>&1; tail -1 $D/smoke.log
python bench.py --steps 20 --warmup 5 > $D/bench_default.json 2> $D/bench_default.err; echo "bench rc=$?"
python bench.py --impl reference --steps 20 --warmup 5 > $D/bench_reference.json 2> $D/bench_reference.err; echo "ref rc=$?"
for cfg in c1 c2 c3 q2 bump c4b c5; do python bench.py --config $cfg --steps 20 --warmup 5 --no-cpu > $D/${cfg}_p1.json 2> $D/${cfg}_p1.err; done
for P in 2 3 4; do for cfg in c4 c4b c5; do
  python -m torch.distributed.run --nnodes=1 --nproc-per-node $P --master-addr 127.0.0.1 --master-port 2969$P bench.py --gpus $P --config $cfg --steps 20 --warmup 5 --no-cpu > $D/${cfg}_p$P.json 2> $D/${cfg}_p$P.err
done; done
SPMAT_HALO=nccl python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29681 bench.py --gpus 2 --steps 20 --warmup 5 --no-cpu --no-e2e > $D/c4_p2_nccl.json 2> $D/c4_p2_nccl.err
SPMAT_HALO=nccl SPMAT_NCCL_MAX_CTAS=0 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29682 bench.py --gpus 2 --steps 20 --warmup 5 --no-cpu --no-e2e > $D/c4_p2_nccl_nocap.json 2> $D/c4_p2_nccl_nocap.err
python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29683 bench.py --impl reference --gpus 4 --steps 5 --warmup 1 > $D/bench_reference_p4.json 2> $D/bench_reference_p4.err
for f in $D/*.json; do python -c "
import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', d.get('launch'), round(d['ms_per_step'],4), round(d['value'],1), (d.get('roofline') or {}).get('frac'), (d.get('e2e') or {}).get('value'), (d.get('clocks') or {}).get('sm_mhz'), (d.get('clocks') or {}).get('reasons'))" 2>/dev/null || (echo "$f failed"; tail -3 ${f%.json}.err); done
python tools/cg_bench.py --configs kuu,bump,bump7 --breakdown --iters 100 > $D/cg_p1.log 2>&1; grep us/iter $D/cg_p1.log
for P in 2 4; do python -m torch.distributed.run --nnodes=1 --nproc-per-node $P --master-addr 127.0.0.1 --master-port 2967$P tools/cg_bench.py --configs kuu,bump --breakdown --iters 100 > $D/cg_p$P.log 2>&1; grep us/iter $D/cg_p$P.log; done
python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29655 tools/sf_bench.py --graph --breakdown > $D/sf_pingpong_graph.log 2>&1; tail -13 $D/sf_pingpong_graph.log
SPMAT_SF=nccl python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29656 tools/sf_bench.py > $D/sf_pingpong_nccl.log 2>&1; tail -13 $D/sf_pingpong_nccl.log
timeout 300 python tools/nvlink_probe.py > $D/nvlink_probe.log 2>&1; tail -2 $D/nvlink_probe.log
