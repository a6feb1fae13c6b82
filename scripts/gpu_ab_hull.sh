cd $GRAFT_REPO_ROOT
for rep in 1 2; do
for so in paper_2208_12737_b200/_lib/variants/*.so; do
  k=$(DRR_B200_LIB=$so timeout 300 python scripts/kbench.py 256 1 2>&1 | tail -1)
  c5=$(DRR_B200_LIB=$so timeout 300 python scripts/c5_modes.py 2>&1 | tail -1)
  echo "$(basename $so) | $k | $c5"
done
done
