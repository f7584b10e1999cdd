#!/bin/bash
# one gpurun call: GPU tests + bench line per SpMV variant (no profiler)
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider 2>&1 | tail -5
CFG=${CFG:-c4}
for k in ${KERNELS:-tma stream}; do
  timeout 300 python bench.py --config $CFG --steps 200 --warmup 10 --no-e2e --no-cpu --kernel $k > gpurun_out/bench_${CFG}_$k.json 2>gpurun_out/bench_${CFG}_$k.err
  python -c "import json;d=json.load(open('gpurun_out/bench_${CFG}_$k.json'));print('$CFG $k', round(d['value'],1), 'GF/s diag', round(d['roofline']['achieved'],1), 'GB/s frac', round(d['roofline']['frac'],3), 'ms', round(d['ms_per_step'],4), d['clocks']['sm_mhz'], d['clocks']['reasons'])" || tail -5 gpurun_out/bench_${CFG}_$k.err
done
