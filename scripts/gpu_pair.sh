OUT=kb4 KB_ARGS="256 32 1" bash scripts/gpu_kb.sh > /dev/null 2>&1
OUT=full3 BENCH_ARGS=--no-cpu-baseline bash scripts/gpu_full.sh
cat gpurun_out/kb4/kbench.json
