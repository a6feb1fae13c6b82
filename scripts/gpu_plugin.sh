# Plugin boundary: the reference's own suites on "cuda" + its dispatcher timed at C2.
cd $GRAFT_REPO_ROOT
O=gpurun_out/${OUT:-plugin}
mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_reference_suite.py tests/test_gpu_parity.py -q > $O/pytest.txt 2>&1
PYTHONPATH=oracle/_ref:.:tests/ref_suite timeout 600 python scripts/plugin_c2.py > $O/plugin_c2.json 2> $O/plugin_c2.err
tail -4 $O/pytest.txt; cat $O/plugin_c2.json; tail -3 $O/plugin_c2.err
