# A/B the variants: parity + kbench per variant .so
cd $GRAFT_REPO_ROOT
for so in paper_2208_12737_b200/_lib/variants/*.so; do
  n=$(basename $so)
  t=$(DRR_B200_LIB=$so timeout 600 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -1)
  k=$(DRR_B200_LIB=$so timeout 300 python scripts/kbench.py 32 2>&1 | tail -1)
  echo "$n | $t | $k"
done
