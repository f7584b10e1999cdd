D=gpurun_out/r02cg; mkdir -p $D
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "cg or graphs or dot" > $D/pytest.log 2>&1; tail -1 $D/pytest.log
for k in 1 2; do python tools/cg_bench.py --configs kuu,bump,bump7 --breakdown --iters 200 > $D/cg_p1_$k.log 2>&1; grep us/iter $D/cg_p1_$k.log; done
MP_CASES=cg python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29641 tests/mp_gpu_parity.py > $D/mp.log 2>&1; grep -E "FAIL|MULTI" $D/mp.log | tail -3
for P in 2 4; do python -m torch.distributed.run --nnodes=1 --nproc-per-node $P --master-addr 127.0.0.1 --master-port 2967$P tools/cg_bench.py --configs kuu,bump --iters 200 > $D/cg_p$P.log 2>&1; grep us/iter $D/cg_p$P.log; done
