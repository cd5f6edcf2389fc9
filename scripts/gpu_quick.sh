cd $GRAFT_REPO_ROOT
export PARPA_DEBUG=1
for p in fused tau; do timeout 60 python scripts/probe.py cfg1 1e5 $p 2>&1 | grep -v Warn | tail -8; done
