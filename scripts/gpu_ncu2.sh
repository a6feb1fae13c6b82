# ncu --set full of the named kernels on scripts/kbench.py (C2, $POSES poses); CSV/detail/SASS exports.
cd $GRAFT_REPO_ROOT
O=gpurun_out/${OUT:-ncu}
mkdir -p $O
for K in ${KERNELS:-k_forward_loss k_forward_jac}; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"^$K\$" -s 1 -c 1 -o /tmp/prof_$K python scripts/kbench.py ${POSES:-32} > $O/ncu_full_$K.log 2>&1
  ncu -i /tmp/prof_$K.ncu-rep --page raw --csv > $O/ncu_full_$K.csv 2>/dev/null
  ncu -i /tmp/prof_$K.ncu-rep --page details > $O/ncu_full_${K}_details.txt 2>/dev/null
  ncu -i /tmp/prof_$K.ncu-rep --page source --csv --print-source sass > $O/ncu_full_${K}_sass.csv 2>/dev/null
done
ls -la $O
