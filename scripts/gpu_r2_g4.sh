cd $GRAFT_REPO_ROOT
O=gpurun_out/g4; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_css.py -x -q --timeout 300 > $O/css.log 2>&1; echo css rc=$?; tail -15 $O/css.log
timeout 900 python -m pytest tests -m gpu -q -x --timeout 300 > $O/pytest_gpu.log 2>&1; echo pytest rc=$?; tail -3 $O/pytest_gpu.log
PARPA_SPROF=1 timeout 120 python scripts/probe_small.py cfg1 1e6 > $O/sprof.log 2>&1; tail -8 $O/sprof.log
timeout 120 python scripts/probe_small.py cfg1 1e6 > $O/small.log 2>&1; cat $O/small.log
