cd $GRAFT_REPO_ROOT
O=gpurun_out/g19; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -x --timeout 300 > $O/pytest.log 2>&1; echo pytest rc=$?; tail -2 $O/pytest.log
for f in ab/libparpa_*.so; do echo "== $f"; for i in 1 2; do PARPA_LIB=$PWD/$f PARPA_SPROF=1 timeout 120 python scripts/probe_small.py cfg1 1e6 2>&1 | grep "sprof" | tail -1; done; PARPA_LIB=$PWD/$f timeout 300 python bench.py --config cfg1 --no-e2e --no-cpu 2>&1 | grep -o '"ms_per_step": [0-9.]*'; done
