# A/B the variants by kernel micro-bench only (no parity): scripts/kbench.py 32
cd $GRAFT_REPO_ROOT
for rep in 1 2; do
for so in paper_2208_12737_b200/_lib/variants/*.so; do
  k=$(DRR_B200_LIB=$so timeout 300 python scripts/kbench.py 32 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read())['32']; print('fwd %.3f fj %.3f bwd %.3f' % (d['fwd_ms'], d['fwd_jac_ms'], d['bwd_ms']))")
  echo "$(basename $so) | $k"
done
done
