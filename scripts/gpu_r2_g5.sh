cd $GRAFT_REPO_ROOT
O=gpurun_out/g5; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_workspace.py tests/test_gpu_css.py -x -q --timeout 300 > $O/new.log 2>&1; echo new rc=$?; tail -15 $O/new.log
timeout 900 python -m pytest tests -m gpu -q -x --timeout 300 > $O/pytest_gpu.log 2>&1; echo pytest rc=$?; tail -3 $O/pytest_gpu.log
PARPA_SPROF=1 timeout 120 python scripts/probe_small.py cfg1 1e6 > $O/sprof.log 2>&1; tail -3 $O/sprof.log
timeout 300 python bench.py --config cfg1 --no-e2e --no-cpu > $O/cfg1.log 2>&1; grep -o '"ms_per_step": [0-9.]*' $O/cfg1.log
bash scripts/ab_bench.sh "yelp taxi" > $O/ab.log 2>&1; cat $O/ab.log
