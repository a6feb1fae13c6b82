cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r02_base
O=gpurun_out/r02_base
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/gpuinfo.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q -rf -x > $O/pytest_gpu.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1
timeout 900 python bench.py --steps 50 --no-cpu-baseline > $O/bench.json 2> $O/bench.err
tail -3 $O/pytest_gpu.txt; cat $O/smoke.txt; cat $O/bench.json; tail -3 $O/bench.err
