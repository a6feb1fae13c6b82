cd $GRAFT_REPO_ROOT
O=gpurun_out/fusedchk
md5sum paper_2208_12737_b200/_lib/libdrr_b200.so
mkdir -p $O

timeout 1800 compute-sanitizer --tool racecheck --print-limit 5 python -m pytest tests/test_gpu_fused_loss.py tests/test_gpu_registration.py -q -x -k "f64_vs_oracle or batch_invariance or three_launch" > $O/racecheck.txt 2>&1
echo "racecheck rc=$?" >> $O/racecheck.txt; tail -3 $O/racecheck.txt
timeout 1800 compute-sanitizer --tool memcheck --leak-check no --print-limit 5 python -m pytest tests/test_gpu_fused_loss.py tests/test_gpu_registration.py -q -x -k "f64_vs_oracle or batch_invariance or three_launch or chains_agree" > $O/memcheck.txt 2>&1
echo "memcheck rc=$?" >> $O/memcheck.txt; tail -3 $O/memcheck.txt
timeout 300 python scripts/kbench.py 256 1 > $O/kbench.json 2>&1; tail -1 $O/kbench.json
timeout 300 python scripts/c3_modes.py 2>&1 | tail -1
