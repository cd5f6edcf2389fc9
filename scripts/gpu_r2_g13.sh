cd $GRAFT_REPO_ROOT
O=gpurun_out/g13; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -x --timeout 300 > $O/pytest.log 2>&1; echo pytest rc=$?; tail -2 $O/pytest.log
PARPA_EMIT_K=4 timeout 900 python -m pytest tests -m gpu -q -x --timeout 300 > $O/pytest_k4.log 2>&1; echo pytest-k4 rc=$?; tail -2 $O/pytest_k4.log
PARPA_EMIT_K=1 timeout 900 python -m pytest tests -m gpu -q -x --timeout 300 > $O/pytest_k1.log 2>&1; echo pytest-k1 rc=$?; tail -2 $O/pytest_k1.log
