cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for w in yelp taxi; do PARPA_DEBUG=1 timeout 120 python scripts/probe2.py $w 2e9 2>&1 | grep -E "per-CTA|GB" | tail -3; done
