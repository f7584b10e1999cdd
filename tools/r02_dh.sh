D=gpurun_out/r02dh; mkdir -p $D
timeout 1500 python -m pytest tests/test_gpu_multirank.py -q -x -p no:cacheprovider -k "parity or tails or lanes" > $D/pytest.log 2>&1; tail -3 $D/pytest.log; grep -E "FAIL" $D/pytest.log | head
for P in 2 4; do python -m torch.distributed.run --nnodes=1 --nproc-per-node $P --master-addr 127.0.0.1 --master-port 2967$P tools/cg_bench.py --configs kuu --breakdown --iters 200 > $D/cg_p$P.log 2>&1; grep us/iter $D/cg_p$P.log; done
for P in 2 4; do SPMAT_SPMV_KERNEL=tma python -m torch.distributed.run --nnodes=1 --nproc-per-node $P --master-addr 127.0.0.1 --master-port 2966$P tools/cg_bench.py --configs kuu --breakdown --iters 200 > $D/cg_p${P}_tma.log 2>&1; grep us/iter $D/cg_p${P}_tma.log; done
