# A/B library variants (paper_2208_12737_b200/_lib/variants/*.so) with scripts/kbench.py;
# optional TESTVAR=<name>: also run the GPU suite against that variant.
cd $GRAFT_REPO_ROOT
if [ -n "$TESTVAR" ]; then
  DRR_B200_LIB=paper_2208_12737_b200/_lib/variants/$TESTVAR.so timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
fi
for rep in 1 2; do
for so in paper_2208_12737_b200/_lib/variants/*.so; do
  k=$(DRR_B200_LIB=$so timeout 300 python scripts/kbench.py ${KB_ARGS:-256 1} 2>&1 | tail -1)
  echo "$(basename $so) | $k"
done
done
