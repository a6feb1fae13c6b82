cd $GRAFT_REPO_ROOT
OUT=ncu256f POSES=256 KERNELS="k_forward_jac k_forward_loss" bash scripts/gpu_ncu2.sh > /dev/null 2>&1
O=gpurun_out/ncu256f
timeout 1800 compute-sanitizer --tool racecheck --print-limit 5 python -m pytest tests/test_gpu_fused_loss.py -q -x -k "f64_vs_oracle or batch_invariance" > $O/racecheck.txt 2>&1
echo "racecheck rc=$?" >> $O/racecheck.txt
tail -3 $O/racecheck.txt; ls $O
