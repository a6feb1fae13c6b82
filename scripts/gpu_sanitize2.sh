# compute-sanitizer memcheck + racecheck + synccheck over the round-2 kernels:
# the fused loss walk (last-warp counter), its reduction + registration step,
# the two-pass loss, volume pack / bounds / hull, signatures, trimming.
cd $GRAFT_REPO_ROOT
O=gpurun_out/sanitize2
mkdir -p $O
T="tests/test_gpu_fused_loss.py tests/test_gpu_volume_pack.py tests/test_gpu_trim.py tests/test_gpu_fd.py"
K="not c2_trimmed and not bright_low and not reference"
timeout 1800 compute-sanitizer --tool memcheck --leak-check no --print-limit 20 \
  python -m pytest $T -q -x -k "$K" > $O/memcheck.txt 2>&1
echo "memcheck rc=$?" >> $O/memcheck.txt
timeout 1800 compute-sanitizer --tool racecheck --print-limit 20 \
  python -m pytest tests/test_gpu_fused_loss.py tests/test_gpu_trim.py -q -x -k "f64_vs_oracle or batch_invariance or air_inside or hull_matches" > $O/racecheck.txt 2>&1
echo "racecheck rc=$?" >> $O/racecheck.txt
timeout 1800 compute-sanitizer --tool synccheck --print-limit 20 \
  python -m pytest tests/test_gpu_fused_loss.py tests/test_gpu_registration.py -q -x -k "f64_vs_oracle or three_launch or image_loss" > $O/synccheck.txt 2>&1
echo "synccheck rc=$?" >> $O/synccheck.txt
for f in memcheck racecheck synccheck; do tail -4 $O/$f.txt; done
