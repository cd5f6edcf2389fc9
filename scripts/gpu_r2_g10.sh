cd $GRAFT_REPO_ROOT
for i in 1 2; do
  timeout 300 python -m pytest tests/test_gpu_css.py -q -x --timeout 300 -k "taxi" 2>&1 | tail -2
  PARPA_EMIT_K=1 timeout 300 python -m pytest tests/test_gpu_css.py -q -x --timeout 300 -k "taxi" 2>&1 | tail -2
  PARPA_LIB=$PWD/ab/libparpa_a_head.so timeout 300 python -m pytest tests/test_gpu_css.py -q -x --timeout 300 -k "taxi" 2>&1 | tail -2
done
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x --timeout 300 -k "taxi" 2>&1 | tail -3
