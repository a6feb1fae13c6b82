# compute-sanitizer memcheck over the kernels added last in round 2: per-ray
# signatures (fd.ray_fd_report), the explicit-ray tangent epilogue
# (drr_raysum_tangents) and the >65535-pose chunking of loss_and_gradient.
cd $GRAFT_REPO_ROOT
O=gpurun_out/sanitize3
mkdir -p $O
timeout 1800 compute-sanitizer --tool memcheck --leak-check no --print-limit 20 \
  python -m pytest tests/test_gpu_fd.py tests/test_gpu_parity.py -q -x \
  -k "ray_signatures or ray_fd_small or raysum_tangents or beyond_one_launch or kernel_cases" \
  > $O/memcheck.txt 2>&1
echo "memcheck rc=$?" >> $O/memcheck.txt
tail -4 $O/memcheck.txt
