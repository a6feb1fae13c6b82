# compute-sanitizer memcheck + racecheck over the small parity cases
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
SEL="kernel_cases or random_rays or clip or pose_renders or backward_vs_oracle or forward_jac_matches or batched_equals or blob_and_corner or beyond_one_launch"
timeout 1500 compute-sanitizer --tool memcheck --leak-check no --print-limit 20 \
  python -m pytest tests/test_gpu_parity.py -q -x -k "$SEL" > gpurun_out/sanitize_memcheck.txt 2>&1
echo "memcheck rc=$?" >> gpurun_out/sanitize_memcheck.txt
timeout 1500 compute-sanitizer --tool racecheck --print-limit 20 \
  python -m pytest tests/test_gpu_parity.py -q -x -k "kernel_cases or pose_renders or backward_vs_oracle or forward_jac_matches" > gpurun_out/sanitize_racecheck.txt 2>&1
echo "racecheck rc=$?" >> gpurun_out/sanitize_racecheck.txt
tail -5 gpurun_out/sanitize_memcheck.txt; tail -5 gpurun_out/sanitize_racecheck.txt
