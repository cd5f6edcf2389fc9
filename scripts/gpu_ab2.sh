cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?; tail -1 gpurun_out/smoke.log
timeout 600 python -m pytest tests -m gpu -q -x --timeout 120 > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/pytest_gpu.log
for v in A C; do
  if [ $v = A ]; then unset PARPA_LIB; else export PARPA_LIB=$PWD/abtest/lib$v.so; fi
  for w in yelp taxi clf cfg1; do echo -n "$v "; timeout 120 python scripts/probe2.py $w 2e9 2>&1 | grep -E "into|Error" | tail -1; done
done
