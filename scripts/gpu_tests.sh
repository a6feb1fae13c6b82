cd $GRAFT_REPO_ROOT
O=gpurun_out/${OUT:-tests}
mkdir -p $O
timeout 1500 python -m pytest ${TESTS:-tests} -m gpu -q -rf > $O/pytest_gpu.txt 2>&1
grep -E "passed|failed|FAILED|Error|^E  " $O/pytest_gpu.txt | tail -30
