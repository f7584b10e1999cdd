#!/bin/bash
# one gpurun call: tests, bench variants, launch list, ncu full on the top kernel
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider 2>&1 | tail -15
for k in tma stream vector; do
  timeout 300 python bench.py --steps 200 --warmup 10 --no-e2e --no-cpu --kernel $k > gpurun_out/bench_$k.json 2>gpurun_out/bench_$k.err
  python -c "import json;d=json.load(open('gpurun_out/bench_$k.json'));print('$k', round(d['value'],1), 'GF/s', round(d['roofline']['achieved'],1), 'GB/s frac', round(d['roofline']['frac'],3), d['clocks'])" || tail -5 gpurun_out/bench_$k.err
done
timeout 300 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_launch.log 2>&1
echo "launch list rc=$?"
timeout 300 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/plain2.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_spmv_tma -s 2 -c 1 -o gpurun_out/prof_tma python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_full.log 2>&1
echo "ncu full rc=$?"
