# One ncu --set full capture of $NCU_KERNEL (default k_forward_jac) on scripts/kbench.py 32,
# exported on the box (details page + raw CSV); the .ncu-rep stays in /tmp.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
K=${NCU_KERNEL:-k_forward_jac}
T=${NCU_TAG:-iter}
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"^$K\$" -s 2 -c 1 -o /tmp/prof_$K python scripts/kbench.py 32 > gpurun_out/ncu_${T}_$K.log 2>&1
ncu -i /tmp/prof_$K.ncu-rep --page raw --csv > gpurun_out/ncu_${T}_$K.csv 2>/dev/null
ncu -i /tmp/prof_$K.ncu-rep --page details > gpurun_out/ncu_${T}_${K}_details.txt 2>/dev/null
tail -2 gpurun_out/ncu_${T}_$K.log
