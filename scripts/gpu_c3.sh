cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_registration.py tests/test_gpu_fused_loss.py tests/test_gpu_api.py tests/test_gpu_acceptance.py -m gpu -q -rf 2>&1 | tail -4
timeout 300 python scripts/c3_modes.py
