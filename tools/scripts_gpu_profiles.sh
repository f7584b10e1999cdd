#!/bin/bash
# refresh the committed evidence: smoke, default bench line, launch list, ncu --set full of
# the hot kernel for C4 (CSR), C3 (CSR, Q1 element COO) and C5 (3x3 block-CSR)
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 600 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "bench rc=$?"
CMD="python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu"
timeout 300 $CMD > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/launches_c4.csv $CMD > gpurun_out/ncu_launch.log 2>&1
echo "launch list rc=$?"
for spec in "c4:k_spmv_tma:1" "c3:k_spmv_tma:1" "c5:k_spmv_bsr3:3"; do
  IFS=: read CFG K BS <<< "$spec"
  CMD="python bench.py --config $CFG --block-size $BS --steps 5 --warmup 3 --no-e2e --no-cpu"
  timeout 600 $CMD > gpurun_out/plain_$CFG.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -s 2 -c 1 -o gpurun_out/prof_final_$CFG $CMD > gpurun_out/ncu_$CFG.log 2>&1
  echo "ncu $CFG rc=$?"
done
