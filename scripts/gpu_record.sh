# A full record run: tests, smoke, bench (with the CPU baseline), the reference
# arm, the 2-rank shared-GPU bench, the ncu launch list, single-pose K A/B.
cd $GRAFT_REPO_ROOT
O=gpurun_out/${OUT:-record}
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/gpuinfo.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -rf > $O/pytest_gpu.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1
timeout 1200 python bench.py > $O/bench.json 2> $O/bench.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_ref.json 2> $O/bench_ref.err
DRR_BENCH_SHARED_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 10 --no-cpu-baseline \
  > $O/bench_2ranks_shared.json 2> $O/bench_2ranks_shared.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_" -c 60 --csv --log-file $O/ncu_launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-other-configs > $O/ncu_bench.log 2>&1
timeout 300 python scripts/kbench_split.py > $O/kbench_split.json 2> $O/kbench_split.err
grep -E "passed|failed|FAILED" $O/pytest_gpu.txt | tail -5; cat $O/smoke.txt; cut -c1-400 $O/bench.json; tail -2 $O/bench.err; cat $O/bench_ref.json; tail -2 $O/bench_ref.err; cut -c1-300 $O/bench_2ranks_shared.json; tail -2 $O/bench_2ranks_shared.err; cat $O/kbench_split.json
