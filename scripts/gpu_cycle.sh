# One GPU cycle: all -m gpu tests, smoke, bench (N=1, no CPU leg unless CPU=1),
# the population study, and kbench.  Outputs under gpurun_out/$OUT.
cd $GRAFT_REPO_ROOT
O=gpurun_out/${OUT:-cycle}
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -rf > $O/pytest_gpu.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1
if [ "$CPU" = "1" ]; then BA=""; else BA="--no-cpu-baseline"; fi
timeout 1200 python bench.py --steps ${STEPS:-30} $BA > $O/bench.json 2> $O/bench.err
if [ -n "$POP" ]; then timeout 900 python scripts/population_study.py --n $POP > $O/population.json 2> $O/population.err; fi
timeout 300 python scripts/kbench.py 256 32 1 > $O/kbench.json 2> $O/kbench.err
grep -E "passed|failed|FAILED|Error" $O/pytest_gpu.txt | tail -12; cat $O/smoke.txt; cut -c1-600 $O/bench.json; tail -3 $O/bench.err; cat $O/population.json 2>/dev/null; tail -2 $O/population.err 2>/dev/null; cat $O/kbench.json
