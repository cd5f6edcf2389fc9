cd $GRAFT_REPO_ROOT
for w in yelp taxi; do timeout 120 python scripts/probe2.py $w 2e9 2>&1 | grep -E "GB|Error" | tail -3; done
export PARPA_DEBUG=1
for w in yelp; do timeout 120 python scripts/probe.py $w 1e9 fused 2>&1 | grep -E "per-CTA|ok|MISMATCH|Error" | tail -3; done
