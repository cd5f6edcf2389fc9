cd $GRAFT_REPO_ROOT
O=gpurun_out/g17; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -x --timeout 300 > $O/pytest.log 2>&1; echo pytest rc=$?; tail -2 $O/pytest.log
bash scripts/ab_bench.sh "yelp clf taxi" > $O/ab.log 2>&1; cat $O/ab.log
