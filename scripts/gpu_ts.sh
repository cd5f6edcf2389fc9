cd $GRAFT_REPO_ROOT
for w in yelp taxi clf cfg1; do timeout 120 python scripts/probe2.py $w 2e9 2>&1 | grep -E "into|Error" | tail -1; done
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e --timestamps 2>&1 | tail -1
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 --timestamps 2>&1 | tail -1
