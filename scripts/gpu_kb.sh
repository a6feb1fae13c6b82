cd $GRAFT_REPO_ROOT
O=gpurun_out/${OUT:-kb}
mkdir -p $O
timeout 300 python scripts/kbench.py ${KB_ARGS:-256 32 1} > $O/kbench.json 2> $O/kbench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_" -c 40 --csv --log-file $O/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-other-configs > $O/ncu_bench.log 2>&1
cat $O/kbench.json; tail -3 $O/kbench.err
python - <<PY
import csv,collections
rows=[r for r in csv.reader(open("$O/launches.csv")) if len(r)>10]
hdr=rows[0]; ki=hdr.index("Kernel Name"); vi=hdr.index("Metric Value")
for r in rows[1:]:
    print(r[ki][:60], r[vi])
PY
