# Variant A/B (scripts/gpu_ab_var.sh) plus the C5 chain A/B (stored Jacobian vs fused walk).
cd $GRAFT_REPO_ROOT
bash scripts/gpu_ab_var.sh
echo "c5 | $(timeout 600 python scripts/c5_modes.py 2>&1 | tail -1)"
