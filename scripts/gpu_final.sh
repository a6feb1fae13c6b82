# Round-end confirmation at HEAD: the TMA tail's new tiles test under memcheck
# and synccheck first (short timeouts), then the full record run.
cd $GRAFT_REPO_ROOT
O=gpurun_out/${OUT:-final}
mkdir -p $O
timeout 300 python -m pytest tests/test_gpu_fused_loss.py -q -k "tma_path" > $O/tma_test.txt 2>&1; tail -1 $O/tma_test.txt
for tool in memcheck synccheck; do
  timeout 600 compute-sanitizer --tool $tool --print-limit 5 python -m pytest tests/test_gpu_fused_loss.py -q -k "tma_path" > $O/sanitize_tma_$tool.txt 2>&1; tail -1 $O/sanitize_tma_$tool.txt
done
OUT=${OUT:-final} bash scripts/gpu_record.sh
