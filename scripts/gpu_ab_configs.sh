# A/B the variants on C1/C4/C5 (scripts/kbench_configs.py)
cd $GRAFT_REPO_ROOT
for so in paper_2208_12737_b200/_lib/variants/*.so; do
  echo "$(basename $so) | $(DRR_B200_LIB=$so timeout 300 python scripts/kbench_configs.py 2>&1 | tail -1)"
done
