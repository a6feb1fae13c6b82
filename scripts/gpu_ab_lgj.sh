# A/B of library variants on the loss + contraction tail: kbench (256 C2 poses) and C5's chains.
cd $GRAFT_REPO_ROOT
for rep in 1 2; do
for so in paper_2208_12737_b200/_lib/variants/*.so; do
  k=$(DRR_B200_LIB=$so timeout 300 python scripts/kbench.py 256 2>&1 | tail -1)
  c=$(DRR_B200_LIB=$so timeout 300 python scripts/c5_modes.py 2>&1 | tail -1)
  echo "$(basename $so) | $k | $c"
done
done
