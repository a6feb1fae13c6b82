# The launch-time TMA / register choice of k_loss_grad_jac: bitwise against
# the register-only build, the fused-loss tests, timing at 256 and 32 poses.
cd $GRAFT_REPO_ROOT
O=gpurun_out/lgj_check
mkdir -p $O
V=paper_2208_12737_b200/_lib/variants
timeout 300 python scripts/lgj_dump.py $O/main.npz > /dev/null
DRR_B200_LIB=$V/b_notma.so timeout 300 python scripts/lgj_dump.py $O/notma.npz > /dev/null
python -c "
import numpy as np
a=np.load('$O/main.npz'); b=np.load('$O/notma.npz')
print({k: bool(np.array_equal(a[k], b[k])) for k in a.files})"
timeout 900 python -m pytest tests/test_gpu_fused_loss.py -q 2>&1 | tail -2
for rep in 1 2; do
  echo "main | $(timeout 300 python scripts/kbench.py 256 32 2>&1 | tail -1)"
  echo "notma | $(DRR_B200_LIB=$V/b_notma.so timeout 300 python scripts/kbench.py 256 32 2>&1 | tail -1)"
done
