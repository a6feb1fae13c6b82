# A/B library variants x trimming modes with scripts/kbench.py (256 poses and 1 pose)
cd $GRAFT_REPO_ROOT
for rep in 1 2; do
for so in paper_2208_12737_b200/_lib/variants/*.so; do
  for m in ${MODES:-box hull}; do
    k=$(DRR_B200_LIB=$so DRR_KBENCH_TRIM=$m timeout 300 python scripts/kbench.py 256 1 2>&1 | tail -1)
    echo "$(basename $so) $m | $k"
  done
done
done
