# quick iteration: parity tests + kernel micro-bench + bench line
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -rf -x > gpurun_out/pytest_gpu.txt 2>&1
timeout 300 python scripts/kbench.py 32 1 > gpurun_out/kbench.json 2> gpurun_out/kbench.err
timeout 600 python bench.py --steps 50 --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err
tail -15 gpurun_out/pytest_gpu.txt; cat gpurun_out/kbench.json; tail -3 gpurun_out/kbench.err; cat gpurun_out/bench.json; tail -3 gpurun_out/bench.err
