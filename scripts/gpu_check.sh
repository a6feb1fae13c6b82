# Full round check: parity, smoke, bench (+ reference arm), ncu launch list and full captures.
# The .ncu-rep files are exported to CSV on the box and removed (gpurun_out/ merges back <= 64 MiB).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpuinfo.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q -rf > gpurun_out/pytest_gpu.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 300 python scripts/kbench.py 32 1 > gpurun_out/kbench.json 2> gpurun_out/kbench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_" -c 60 --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-other-configs > gpurun_out/ncu_bench.log 2>&1
for K in k_forward_jac k_forward; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"^$K\$" -s 2 -c 1 -o /tmp/prof_$K python scripts/kbench.py 32 > gpurun_out/ncu_full_$K.log 2>&1
  ncu -i /tmp/prof_$K.ncu-rep --page raw --csv > gpurun_out/ncu_full_$K.csv 2>/dev/null
  ncu -i /tmp/prof_$K.ncu-rep --page details > gpurun_out/ncu_full_${K}_details.txt 2>/dev/null
  ncu -i /tmp/prof_$K.ncu-rep --page source --csv --print-source sass > gpurun_out/ncu_full_${K}_sass.csv 2>/dev/null
done
tail -3 gpurun_out/pytest_gpu.txt; cat gpurun_out/smoke.txt; cat gpurun_out/bench.json; tail -3 gpurun_out/bench.err; cat gpurun_out/bench_ref.json; tail -3 gpurun_out/bench_ref.err
