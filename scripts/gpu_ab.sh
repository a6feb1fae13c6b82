# A/B the walk variants: parity on the default build, then kbench per variant .so
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -x -rf > gpurun_out/pytest_gpu.txt 2>&1
tail -2 gpurun_out/pytest_gpu.txt
echo "default: $(timeout 300 python scripts/kbench.py 32 1 2>&1 | tail -1)"
for so in paper_2208_12737_b200/_lib/variants/*.so; do
  echo "$(basename $so): $(DRR_B200_LIB=$so timeout 300 python scripts/kbench.py 32 1 2>&1 | tail -1)"
done
