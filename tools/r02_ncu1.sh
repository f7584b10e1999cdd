# 1 GPU: ncu --set full of the COO numeric kernels (C3 element COO, C5 3x3 direct), the pure dot (bump CG)
D=gpurun_out/r02ncu1; mkdir -p $D
C3="python bench.py --config c3 --steps 5 --warmup 3 --no-e2e --no-cpu"
C5="python bench.py --config c5 --steps 5 --warmup 3 --no-e2e --no-cpu"
CG="python tools/cg_bench.py --configs bump --iters 20"
timeout 600 $C3 > $D/plain_c3.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_numeric -s 1 -c 1 -o $D/prof_c3_numeric $C3 > $D/ncu_c3.log 2>&1; echo "c3 rc=$?"
timeout 600 $C5 > $D/plain_c5.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_numeric -s 1 -c 1 -o $D/prof_c5_numeric $C5 > $D/ncu_c5.log 2>&1; echo "c5 rc=$?"
timeout 600 $CG > $D/plain_cg.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_dot_partial -s 5 -c 1 -o $D/prof_dot $CG > $D/ncu_dot.log 2>&1; echo "dot rc=$?"
grep -h set_values $D/plain_c3.log | head -2
