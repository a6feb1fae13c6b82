# A/B + parity of the TMA-staged k_loss_grad_jac: every variant in
# paper_2208_12737_b200/_lib/variants (b_notma = the register-staged form) is
# compared bitwise against b_notma, then timed (kbench 256 / 32 poses, C5 chains).
cd $GRAFT_REPO_ROOT
O=gpurun_out/lgj_tma
mkdir -p $O
V=paper_2208_12737_b200/_lib/variants
for so in $V/*.so; do v=$(basename $so .so); DRR_B200_LIB=$so timeout 300 python scripts/lgj_dump.py $O/$v.npz > /dev/null; done
python -c "
import glob, numpy as np
ref=np.load('$O/b_notma.npz')
for f in sorted(glob.glob('$O/*.npz')):
    a=np.load(f); print(f.split('/')[-1], all(np.array_equal(a[k], ref[k]) for k in ref.files))"
if [ -z "$NOTEST" ]; then
DRR_B200_LIB=$V/a_tma.so timeout 900 python -m pytest tests/test_gpu_fused_loss.py tests/test_gpu_registration.py tests/test_gpu_distributed.py tests/test_gpu_api.py -q 2>&1 | tail -2
for tool in memcheck racecheck synccheck; do
  DRR_B200_LIB=$V/a_tma.so timeout 900 compute-sanitizer --tool $tool --print-limit 5 python -m pytest tests/test_gpu_fused_loss.py -q -k "loss_grad_jac" > $O/$tool.txt 2>&1; tail -1 $O/$tool.txt
done
fi
for rep in 1 2; do for so in $V/*.so; do
  k=$(DRR_B200_LIB=$so timeout 300 python scripts/kbench.py 256 32 2>&1 | tail -1)
  c=$(DRR_B200_LIB=$so timeout 300 python scripts/c5_modes.py 2>&1 | tail -1)
  echo "$(basename $so) | $k | $c"
done; done
