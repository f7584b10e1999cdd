# 1-GPU check: new GPU tests, default bench line, smoke
D=gpurun_out/r02g1; mkdir -p $D
timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -rA -q -p no:cacheprovider -k "full_size or every_row or block_csr or cuda_graphs" > $D/pytest.log 2>&1; tail -12 $D/pytest.log
python bench.py --steps 20 --warmup 5 > $D/bench.json 2> $D/bench.err; tail -c 3000 $D/bench.json; tail -5 $D/bench.err
python bench.py --impl reference --steps 20 --warmup 5 > $D/ref.json 2> $D/ref.err; cat $D/ref.json; tail -3 $D/ref.err
