cd $GRAFT_REPO_ROOT
for n in 1e9 4.8e9; do
  for p in count tau fused plan; do timeout 120 python scripts/probe.py yelp $n $p 2>&1 | grep -v Warn | tail -2; done
done
