cd $GRAFT_REPO_ROOT
O=gpurun_out/g6; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -x --timeout 300 > $O/pytest_gpu.log 2>&1; echo pytest rc=$?; tail -3 $O/pytest_gpu.log
bash scripts/ab_bench.sh "yelp taxi clf" > $O/ab.log 2>&1; cat $O/ab.log
