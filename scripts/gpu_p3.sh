cd $GRAFT_REPO_ROOT
for w in yelp taxi; do timeout 120 python scripts/probe3.py $w 2e9 2>&1 | tail -2; done
