# Round-2 ncu evidence on 1 GPU: launch list of the default bench command, ncu --set full of the hot kernels
D=gpurun_out/r02ncu; mkdir -p $D
CMD="python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e"
timeout 600 $CMD > $D/plain.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file $D/launches_c4.csv $CMD > $D/ncu_launch.log 2>&1; echo "launch list rc=$?"
for spec in "c4:k_spmv_tma:2" "c5:k_spmv_bsr3:2" "c1:k_spmv_direct:2" "c4:k_numeric:1" "bump:k_spmv_tma:2" "c3:k_spmv_tma:2" "c3:k_numeric:1"; do
  IFS=: read CFG K S <<< "$spec"
  CMD="python bench.py --config $CFG --steps 5 --warmup 3 --no-e2e --no-cpu"
  timeout 600 $CMD > $D/plain_$CFG.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -s $S -c 1 -o $D/prof_${CFG}_$K $CMD > $D/ncu_${CFG}_$K.log 2>&1
  echo "ncu $CFG $K rc=$?"
done
