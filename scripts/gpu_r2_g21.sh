cd $GRAFT_REPO_ROOT
O=gpurun_out/g21; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -x --timeout 300 > $O/pytest.log 2>&1; echo pytest rc=$?; tail -2 $O/pytest.log
for f in ab/libparpa_*.so; do echo "== $f"; PARPA_LIB=$PWD/$f PARPA_SPROF=1 timeout 120 python scripts/probe_small.py cfg1 1e6 2>&1 | grep "sprof" | tail -1; done
bash scripts/ab_bench.sh "clf" > $O/ab.log 2>&1; cat $O/ab.log
