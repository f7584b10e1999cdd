D=gpurun_out/r02cgl; mkdir -p $D
SPMAT_CG_LANES=one timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "cg" > $D/pytest.log 2>&1; tail -1 $D/pytest.log
for rep in 1 2; do for l in own one; do SPMAT_CG_LANES=$l python tools/cg_bench.py --configs kuu --iters 200 > $D/cg_$l.log 2>&1; echo "lanes=$l $(grep us/iter $D/cg_$l.log)"; done; done
