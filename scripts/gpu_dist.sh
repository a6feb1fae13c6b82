# Multi-rank product path on the one-GPU box: the ws2 GPU test, bench at N=1,
# and bench with 2 ranks sharing cuda:0 (gloo; DRR_BENCH_SHARED_GPU=1).
cd $GRAFT_REPO_ROOT
O=gpurun_out/${OUT:-dist}
mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_distributed.py -m gpu -q -rf -x > $O/pytest_dist.txt 2>&1
timeout 900 python bench.py --steps 30 ${BENCH_ARGS} > $O/bench1.json 2> $O/bench1.err
DRR_BENCH_SHARED_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 10 --no-cpu-baseline \
  > $O/bench2.json 2> $O/bench2.err
tail -5 $O/pytest_dist.txt; cat $O/bench1.json; tail -5 $O/bench1.err; cat $O/bench2.json; tail -5 $O/bench2.err
