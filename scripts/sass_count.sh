# usage: bash scripts/sass_count.sh [-Dmacro ...]  -> fast-path instruction counts of the walk loops
cd "$(dirname "$0")/.."
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo --fmad=false -std=c++17 -cubin -Xptxas=-v "$@" \
  -o /tmp/harness.cubin scripts/sass_harness.cu > /tmp/harness.log 2>&1 || { grep -i error /tmp/harness.log; exit 1; }
grep -A2 "Compiling entry.*k_\(forward\|backward\)" /tmp/harness.log | grep "Used\|spill"
cuobjdump -sass /tmp/harness.cubin > /tmp/harness.sass
python3 scripts/sass_fastpath.py /tmp/harness.sass | grep "k_forward\|k_backward"
