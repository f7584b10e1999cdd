D=gpurun_out/r02bsrc; mkdir -p $D
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "block_csr or full_size or numeric" > $D/pytest.log 2>&1; tail -1 $D/pytest.log
MP_CASES=elasticity,full-c5 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29641 tests/mp_gpu_parity.py > $D/mp.log 2>&1; grep -E "FAIL|MULTI" $D/mp.log | tail -3
