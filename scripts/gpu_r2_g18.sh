cd $GRAFT_REPO_ROOT
O=gpurun_out/g18; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -x --timeout 300 > $O/pytest.log 2>&1; echo pytest rc=$?; tail -2 $O/pytest.log
PARPA_EMIT_K=4 timeout 900 python -m pytest tests -m gpu -q -x --timeout 300 > $O/pytest_k4.log 2>&1; echo pytest-k4 rc=$?; tail -2 $O/pytest_k4.log
bash scripts/ab_bench.sh "clf yelp" > $O/ab.log 2>&1; cat $O/ab.log
