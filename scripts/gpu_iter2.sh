cd $GRAFT_REPO_ROOT
O=gpurun_out/${OUT:-iter2}
mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_distributed.py tests/test_gpu_reference_suite.py -m gpu -q -rf > $O/pytest.txt 2>&1
PYTHONPATH=oracle/_ref:.:tests/ref_suite timeout 600 python scripts/plugin_c2.py > $O/plugin_c2.json 2> $O/plugin_c2.err
tail -60 $O/pytest.txt; cat $O/plugin_c2.json; tail -3 $O/plugin_c2.err
