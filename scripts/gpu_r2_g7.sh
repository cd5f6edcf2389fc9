cd $GRAFT_REPO_ROOT
O=gpurun_out/g7; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -x --timeout 300 > $O/pytest_gpu.log 2>&1; echo pytest rc=$?; tail -5 $O/pytest_gpu.log
PARPA_SPROF=1 timeout 120 python scripts/probe_small.py cfg1 1e6 > $O/sprof.log 2>&1; tail -2 $O/sprof.log
bash scripts/ab_bench.sh "clf taxi yelp cfg1" > $O/ab.log 2>&1; cat $O/ab.log
