# Full round check: parity, smoke, bench (+ reference arm), ncu launch list and full captures.
cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpuinfo.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q -rf > gpurun_out/pytest_gpu.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_" -c 60 --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_forward_jac -s 2 -c 1 -o gpurun_out/prof_fj python scripts/kbench.py 32 > gpurun_out/ncu_full.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'^k_forward$' -s 2 -c 1 -o gpurun_out/prof_fwd python scripts/kbench.py 32 > gpurun_out/ncu_full_fwd.log 2>&1
tail -3 gpurun_out/pytest_gpu.txt; cat gpurun_out/smoke.txt; cat gpurun_out/bench.json; tail -3 gpurun_out/bench.err; cat gpurun_out/bench_ref.json; tail -3 gpurun_out/bench_ref.err
