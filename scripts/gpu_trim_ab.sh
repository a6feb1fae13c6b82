cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_trim.py -m gpu -q -rf 2>&1 | tail -3
for m in none box hull; do echo "$m $(DRR_KBENCH_TRIM=$m timeout 300 python scripts/kbench.py 256 1 2>&1 | tail -1)"; done
