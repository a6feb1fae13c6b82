# quick iteration: parity tests + kernel micro-bench (+ optional ncu of one kernel)
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -rf --durations=8 > gpurun_out/pytest_gpu.txt 2>&1
timeout 300 python scripts/kbench.py 32 1 > gpurun_out/kbench.json 2> gpurun_out/kbench.err
timeout 300 python scripts/bench_registration.py 1 64 > gpurun_out/regbench.json 2> gpurun_out/regbench.err
if [ -n "$NCU_KERNEL" ]; then
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$NCU_KERNEL -s 3 -c 1 -o gpurun_out/prof_iter python scripts/kbench.py 32 > gpurun_out/ncu_iter.log 2>&1
fi
tail -15 gpurun_out/pytest_gpu.txt; cat gpurun_out/kbench.json; cat gpurun_out/regbench.json; tail -3 gpurun_out/regbench.err
