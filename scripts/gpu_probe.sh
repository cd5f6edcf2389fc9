cd $GRAFT_REPO_ROOT
for n in 1e5 1e6 1e7 1e8; do
  for p in count fused plan tau; do timeout 60 python scripts/probe.py yelp $n $p 2>&1 | grep -v Warn | tail -2; done
done
timeout 120 python -m pytest tests/test_gpu_ranges.py -q -x --timeout 60 2>&1 | tail -5
