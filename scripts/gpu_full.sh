# pytest -m gpu (all), smoke, bench (N=1) and the 2-rank shared-GPU bench.
cd $GRAFT_REPO_ROOT
O=gpurun_out/${OUT:-full}
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -rf > $O/pytest_gpu.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1
timeout 900 python bench.py --steps ${STEPS:-30} ${BENCH_ARGS} > $O/bench.json 2> $O/bench.err
if [ -n "$TWO_RANKS" ]; then
DRR_BENCH_SHARED_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 10 --no-cpu-baseline \
  > $O/bench2.json 2> $O/bench2.err
fi
grep -E "passed|failed|FAILED|Error" $O/pytest_gpu.txt | tail -15; cat $O/smoke.txt; cut -c1-1500 $O/bench.json; tail -3 $O/bench.err
