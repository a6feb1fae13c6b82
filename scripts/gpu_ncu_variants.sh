cd $GRAFT_REPO_ROOT
O=gpurun_out/${OUT:-ncuvar}
mkdir -p $O
for so in paper_2208_12737_b200/_lib/variants/*.so; do
  n=$(basename $so .so)
  DRR_B200_LIB=$so DRR_KBENCH_TRIM=${MODE:-box} timeout 900 ncu --set full --clock-control none -k regex:"^k_forward_jac\$" -s 1 -c 1 -o /tmp/p_$n python scripts/kbench.py 32 > $O/$n.log 2>&1
  ncu -i /tmp/p_$n.ncu-rep --page raw --csv > $O/$n.csv 2>/dev/null
done
ls $O
