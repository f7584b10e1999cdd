D=gpurun_out/r02lazy; mkdir -p $D
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "transpose or sf or halo" > $D/pytest.log 2>&1; tail -1 $D/pytest.log
for H in peer nccl; do SPMAT_HALO=$H MP_CASES=stencil,q1,random1,random2,transpose,sf1,sf2,box7-int,elasticity timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29671 tests/mp_gpu_parity.py > $D/mp_$H.log 2>&1; grep -E "FAIL|MULTI" $D/mp_$H.log | tail -3; done
