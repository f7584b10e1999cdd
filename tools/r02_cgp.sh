# One-launch CG for small single-rank matrices: parity (bit-identical to the graph path) and µs/iteration
D=gpurun_out/r02cgp; mkdir -p $D
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "cg" > $D/pytest.log 2>&1; tail -1 $D/pytest.log
for rep in 1 2; do for pp in 1 0; do SPMAT_CG_PERSIST=$pp python tools/cg_bench.py --configs kuu --iters 100 > $D/cg_$pp.log 2>&1; echo "persist=$pp $(grep us/iter $D/cg_$pp.log)"; done; done
SPMAT_CG_PERSIST=1 python tools/cg_bench.py --configs kuu,bump7 --breakdown --iters 400 > $D/cg_long.log 2>&1; grep us/iter $D/cg_long.log
