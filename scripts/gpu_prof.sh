# parity tests + kernel micro-bench + one ncu --set full capture of $NCU_KERNEL
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -rf -x > gpurun_out/pytest_gpu.txt 2>&1
timeout 300 python scripts/kbench.py 32 1 > gpurun_out/kbench.json 2> gpurun_out/kbench.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:${NCU_KERNEL:-k_forward_jac} -s 2 -c 1 -o gpurun_out/prof_${NCU_TAG:-iter} python scripts/kbench.py 32 > gpurun_out/ncu_iter.log 2>&1
tail -4 gpurun_out/pytest_gpu.txt; cat gpurun_out/kbench.json; tail -3 gpurun_out/kbench.err; tail -3 gpurun_out/ncu_iter.log
