#!/bin/bash
# ncu --set full of the diag SpMV kernel variants on C4 (after a clean plain run)
cd $GRAFT_REPO_ROOT
CFG=${CFG:-c4}
for k in ${KERNELS:-tma}; do
  CMD="python bench.py --config $CFG --steps 5 --warmup 3 --no-e2e --no-cpu --kernel $k"
  timeout 300 $CMD > gpurun_out/plain_$k.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_spmv -s 2 -c 1 -o gpurun_out/prof_${CFG}_$k $CMD > gpurun_out/ncu_$k.log 2>&1
  echo "ncu $k rc=$?"
done
