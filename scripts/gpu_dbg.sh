cd $GRAFT_REPO_ROOT
export PARPA_DEBUG=1
for w in yelp taxi; do timeout 120 python scripts/probe.py $w 1e9 fused 2>&1 | grep -E "parpa\]|ok|MISMATCH|Error" | tail -3; done
