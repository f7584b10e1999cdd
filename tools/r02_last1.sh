# Driver-like single-GPU check at the tip, plus an ncu capture of the one-launch CG kernel.
D=gpurun_out/r02last; mkdir -p $D
{ echo "tip: $(cat .tip_sha 2>/dev/null)"; nvidia-smi -L; } > $D/pytest_gpu_1gpu.log
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider >> $D/pytest_gpu_1gpu.log 2>&1; echo "pytest rc=$?"; tail -2 $D/pytest_gpu_1gpu.log
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $D/smoke.log 2>&1; tail -1 $D/smoke.log
timeout 600 ncu --set full --clock-control none -k regex:k_cg_persist -c 1 -o $D/cg_persist python tools/cg_bench.py --configs kuu --iters 50 > $D/ncu_cg.log 2>&1; tail -1 $D/ncu_cg.log
