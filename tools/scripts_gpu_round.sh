#!/bin/bash
# full measurement call: bench line (default), launch list, ncu --set full on the top kernel
cd $GRAFT_REPO_ROOT
CFG=${CFG:-c4}
timeout 600 python bench.py --config $CFG --steps 200 --warmup 10 > gpurun_out/bench_full_$CFG.json 2> gpurun_out/bench_full_$CFG.err
tail -c 3000 gpurun_out/bench_full_$CFG.json
CMD="python bench.py --config $CFG --steps 5 --warmup 3 --no-e2e --no-cpu"
timeout 300 $CMD > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 1000 --csv --log-file gpurun_out/launches_$CFG.csv $CMD > gpurun_out/ncu_launch.log 2>&1
echo "launch list rc=$?"
timeout 300 $CMD > gpurun_out/plain2.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_spmv_tma -s 2 -c 1 -o gpurun_out/prof_full_$CFG $CMD > gpurun_out/ncu_full.log 2>&1
echo "ncu full rc=$?"
