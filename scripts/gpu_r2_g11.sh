cd $GRAFT_REPO_ROOT
echo "== auto"; timeout 300 python -m pytest tests/test_gpu_collab.py tests/test_gpu_css.py -q -x --timeout 300 2>&1 | tail -2
echo "== auto again"; timeout 300 python -m pytest tests/test_gpu_collab.py tests/test_gpu_css.py -q -x --timeout 300 2>&1 | tail -2
echo "== K1"; PARPA_EMIT_K=1 timeout 300 python -m pytest tests/test_gpu_collab.py tests/test_gpu_css.py -q -x --timeout 300 2>&1 | tail -2
echo "== head"; PARPA_LIB=$PWD/ab/libparpa_a_head.so timeout 300 python -m pytest tests/test_gpu_collab.py tests/test_gpu_css.py -q -x --timeout 300 2>&1 | tail -2
echo "== css only"; timeout 300 python -m pytest tests/test_gpu_css.py -q -x --timeout 300 2>&1 | tail -2
echo "== nopdl"; PARPA_NO_PDL=1 timeout 300 python -m pytest tests/test_gpu_collab.py tests/test_gpu_css.py -q -x --timeout 300 2>&1 | tail -2
