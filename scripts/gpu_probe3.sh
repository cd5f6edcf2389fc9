cd $GRAFT_REPO_ROOT
for w in yelp taxi clf; do timeout 120 python scripts/probe2.py $w 2e9 2>&1 | grep -E "GB|Error" | tail -3; done
