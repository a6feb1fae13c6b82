cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpuinfo.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q -rf > gpurun_out/pytest_gpu.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_(forward|backward|reduce)" -c 30 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_backward -s 2 -c 1 -o gpurun_out/prof_bwd python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_forward -s 2 -c 1 -o gpurun_out/prof_fwd python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full_fwd.log 2>&1
ls -la gpurun_out
