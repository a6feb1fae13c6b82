# A/B the library variants in paper_2208_12737_b200/_lib/variants/ with scripts/kbench.py
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/ab
for rep in 1 2; do
for so in paper_2208_12737_b200/_lib/variants/*.so; do
  k=$(DRR_B200_LIB=$so timeout 300 python scripts/kbench.py ${KB_ARGS:-256 32} 2>&1 | tail -1)
  echo "$(basename $so) | $k" | tee -a gpurun_out/ab/ab.txt
done
done
